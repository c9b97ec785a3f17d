"""Host-side mirror of the reference's ``namespace lq`` interface for the W4A8
path, backed by the sm_100a kernels in liblqg.so.

Same names, argument meaning and error behaviour as the reference
(/root/reference/proj/include/lq/gemm.hpp:25-66, bundle.hpp:36-69,
errors.hpp:15-28), so a caller of ``lq::gemm_w4a8_accum`` / ``lq::gemm_w4a8``
can switch to this module and keep its tests. Every compute call runs on the
GPU through the C ABI (include/lqg.h); there is no CPU fallback.

Differences a caller can observe:
  * ``TileConfig`` and ``Engine`` are validated with the reference rules but
    do not change the computation (the reference contract makes results
    independent of both, test_gemm.cpp:96-130).
  * The device layout needs ``group_size % 32 == 0``; other group sizes raise
    ``ValidationError`` at the first GEMM.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib


# ---------------------------------------------------------------- errors
class ValidationError(RuntimeError):
    """lq::ValidationError (errors.hpp:15-17): bad input data."""


class VerificationError(RuntimeError):
    """lq::VerificationError (errors.hpp:19-21): a checked invariant failed."""


class IoError(RuntimeError):
    """lq::IoError (errors.hpp:23-28)."""

    def __init__(self, msg: str, byte_offset: int = 0):
        super().__init__(f"{msg} (byte offset {byte_offset})")
        self.byte_offset = byte_offset


class CudaError(RuntimeError):
    """A CUDA runtime/driver failure inside liblqg (no reference analogue)."""


class UnsupportedDeviceError(RuntimeError):
    """No sm_100 device: liblqg has no CPU fallback."""


_ERRORS = {1: ValidationError, 2: VerificationError, 3: IoError, 4: CudaError, 5: CudaError,
           6: UnsupportedDeviceError}


_OFFSET_RE = None


def check(rc: int) -> None:
    if rc:
        msg = _lib.lib().lqg_last_error().decode()
        if rc == 3:  # "<message> (byte offset N)" -> IoError(message, N), like lq::IoError
            global _OFFSET_RE
            import re
            _OFFSET_RE = _OFFSET_RE or re.compile(r"^(.*) \(byte offset (\d+)\)$", re.S)
            mo = _OFFSET_RE.match(msg)
            if mo:
                raise IoError(mo.group(1), int(mo.group(2)))
        raise _ERRORS.get(rc, RuntimeError)(msg)


# ---------------------------------------------------------------- types
class WeightLayout(enum.IntEnum):
    """bundle.hpp:36-39"""
    PlainRowMajor = 0
    DualMmaPacked = 1


class Engine(enum.IntEnum):
    """gemm.hpp:44"""
    Scalar = 0
    Packed = 1


@dataclass
class FragmentDescriptor:
    """layout.hpp:33-46 (defaults = the Hopper dual-MMA geometry)."""
    warps_per_group: int = 4
    threads_per_warp: int = 32
    mma_m: int = 64
    mma_k: int = 32
    elements_per_thread_per_mma: int = 16
    dual_k_span: int = 64

    def validate(self) -> None:
        """layout.cpp:10-22"""
        slab = self.mma_m * self.mma_k
        per_group = self.warps_per_group * self.threads_per_warp * self.elements_per_thread_per_mma
        if slab != per_group:
            raise ValidationError(f"fragment descriptor mismatch: mma_m*mma_k = {slab} but group "
                                  f"covers {per_group} elements")
        if self.dual_k_span != 2 * self.mma_k:
            raise ValidationError("dual_k_span must be 2*mma_k")
        if 0 in (self.warps_per_group, self.threads_per_warp, self.mma_m, self.mma_k):
            raise ValidationError("fragment descriptor has a zero field")


@dataclass(eq=False)
class QuantizedWeightBundle:
    """bundle.hpp:41-69. Arrays are numpy: packed_weights u8 ((n*k+1)//2),
    group_scales / group_offsets u8 (n*(k//group_size)), channel_scales f32 (n)."""
    n: int = 0
    k: int = 0
    group_size: int = 64
    layout: WeightLayout = WeightLayout.PlainRowMajor
    fragment: FragmentDescriptor = field(default_factory=FragmentDescriptor)
    packed_weights: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    group_scales: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    group_offsets: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    channel_scales: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def groups_per_row(self) -> int:
        return self.k // self.group_size

    def scale_of(self, row: int, group: int) -> int:
        return int(self.group_scales[row * self.groups_per_row() + group])

    def offset_of(self, row: int, group: int) -> int:
        return int(self.group_offsets[row * self.groups_per_row() + group])

    def _view(self):
        """Borrowed lqg_bundle_view; keeps the contiguous arrays alive."""
        keep = [np.ascontiguousarray(self.packed_weights, np.uint8),
                np.ascontiguousarray(self.group_scales, np.uint8),
                np.ascontiguousarray(self.group_offsets, np.uint8),
                np.ascontiguousarray(self.channel_scales, np.float32)]
        f = self.fragment
        v = _lib.BundleViewC(
            self.n, self.k, self.group_size, int(self.layout),
            _lib.FragmentDescriptorC(f.warps_per_group, f.threads_per_warp, f.mma_m, f.mma_k,
                                     f.elements_per_thread_per_mma, f.dual_k_span),
            keep[0].ctypes.data, keep[0].size, keep[1].ctypes.data, keep[2].ctypes.data,
            keep[1].size,
            keep[3].ctypes.data if keep[3].size == self.n else None)
        return v, keep

    def validate(self) -> None:
        """bundle.cpp:89-135 (host-only, same rules and messages)."""
        if self.group_scales.size != self.group_offsets.size:
            raise ValidationError("group parameter arrays have wrong size")
        v, _keep = self._view()
        check(_lib.lib().lqg_bundle_validate(C.byref(v)))

    def prepack(self) -> np.ndarray:
        """The device image of this bundle (host-only, no GPU needed); cache it
        and upload later with DeviceWeights.from_image."""
        if self.group_scales.size != self.group_offsets.size:
            raise ValidationError("group parameter arrays have wrong size")
        nbytes = int(_lib.lib().lqg_image_bytes(self.n, self.k, self.group_size))
        if nbytes == 0:
            raise ValidationError("the sm_100a device layout needs group_size % 32 == 0 (got "
                                  f"{self.group_size})")
        img = np.empty(nbytes, np.uint8)
        v, _keep = self._view()
        check(_lib.lib().lqg_prepack_host(C.byref(v), img.ctypes.data, nbytes))
        return img

    def device_weights(self, device: int = 0) -> "DeviceWeights":
        """A new prepacked device copy of the bundle as it is now (not cached:
        like the reference, every gemm_w4a8 call reads the bundle's current
        arrays; keep the returned handle to reuse an upload)."""
        return DeviceWeights.from_bundle(self, device)


@dataclass
class TileConfig:
    """gemm.hpp:29-33. Validated with the reference rules (gemm.cpp:11-17); the
    device kernel picks its own tiles (results are tile-independent)."""
    m_t: int = 64
    n_t: int = 64
    k_t: int = 64

    def validate(self, b: QuantizedWeightBundle) -> None:
        if self.m_t < 1 or self.n_t < 1 or self.k_t < 1:
            raise ValidationError("tile extents must be >= 1")
        if b.layout == WeightLayout.DualMmaPacked and self.k_t % b.fragment.dual_k_span != 0:
            raise ValidationError(f"k_t must be a multiple of {b.fragment.dual_k_span} when "
                                  "consuming the dual-MMA layout")


@dataclass
class ActivationQuant:
    """gemm.hpp:35-39: values m*k int8 codes in [-127, 127], token_scales m."""
    m: int = 0
    k: int = 0
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int8))
    token_scales: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))


@dataclass
class GemmShape:
    """gemm.hpp:25-27"""
    m: int = 0
    n: int = 0
    k: int = 0


# ---------------------------------------------------------------- entry points
def quantize_activations_per_token(x, m: int, k: int) -> ActivationQuant:
    """gemm.cpp:19-47, computed by the lqg activation-quant kernel (bit-exact)."""
    import torch
    if m < 1 or k < 1:
        raise ValidationError("activation dimensions must be >= 1")
    xa = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).reshape(-1)
    if xa.size != m * k:
        raise ValidationError("activation buffer size does not match m*k")
    dev = torch.device("cuda", torch.cuda.current_device())
    xd = torch.from_numpy(xa).to(dev).view(m, k)
    q, ts = quantize_activations(xd, check_finite=True)
    return ActivationQuant(m, k, q.cpu().numpy().reshape(-1), ts.cpu().numpy())


def _prepare(act: ActivationQuant, weights: QuantizedWeightBundle, tile: TileConfig,
             engine: Engine):
    # gemm.cpp:141-146 and 151-158, in the reference's order
    weights.validate()
    tile.validate(weights)
    if act.k != weights.k:
        raise ValidationError(f"activation depth {act.k} does not match weight depth {weights.k}")
    if act.k * 127 * 127 >= (1 << 31):
        raise ValidationError(f"k = {act.k} risks 32-bit accumulator overflow (k*127*127 >= 2^31)")
    if Engine(engine) == Engine.Packed and tile.k_t % weights.fragment.dual_k_span != 0:
        raise ValidationError(f"k_t must be a multiple of {weights.fragment.dual_k_span} for the "
                              "packed engine")
    vals = np.ascontiguousarray(np.asarray(act.values, dtype=np.int8)).reshape(-1)
    if vals.size != act.m * act.k or act.m < 1:
        raise ValidationError("activation buffer size does not match m*k")
    ts = np.ascontiguousarray(np.asarray(act.token_scales, dtype=np.float32)).reshape(-1)
    import torch
    dw = weights.device_weights(torch.cuda.current_device())
    return dw, vals, ts


def gemm_w4a8_accum(act: ActivationQuant, weights: QuantizedWeightBundle,
                    tile: TileConfig = TileConfig(), engine: Engine = Engine.Packed) -> np.ndarray:
    """gemm.hpp:49-51: INT32 accumulators, row-major m*n (1-D, like the
    reference's std::vector)."""
    dw, vals, _ts = _prepare(act, weights, tile, engine)
    acc = np.empty(act.m * weights.n, np.int32)
    check(_lib.lib().lqg_gemm_w4a8_accum_host(dw.handle, vals.ctypes.data, act.m, acc.ctypes.data,
                                              None))
    return acc


def gemm_w4a8(act: ActivationQuant, weights: QuantizedWeightBundle,
              tile: TileConfig = TileConfig(), engine: Engine = Engine.Packed) -> np.ndarray:
    """gemm.hpp:54-55: float outputs, row-major m*n, bit-identical to the
    reference epilogue (quant.cpp:125-127)."""
    dw, vals, ts = _prepare(act, weights, tile, engine)
    if ts.size != act.m:
        raise ValidationError("token scale array has wrong size")
    y = np.empty(act.m * weights.n, np.float32)
    check(_lib.lib().lqg_gemm_w4a8_host(dw.handle, vals.ctypes.data, ts.ctypes.data, act.m,
                                        y.ctypes.data, 0, None))
    return y


# ---------------------------------------------------------------- device API
Y_DTYPES = {"float32": 0, "float16": 1, "bfloat16": 2}


def _y_code(dtype) -> int:
    name = str(dtype).replace("torch.", "")
    if name not in Y_DTYPES:
        raise ValidationError(f"unsupported output dtype {dtype}")
    return Y_DTYPES[name]


_TORCH = None


def _torch():
    """torch and the dtype objects the launch path compares against, imported
    once (the eager launch path is a few microseconds of host time)."""
    global _TORCH
    if _TORCH is None:
        import torch
        _TORCH = (torch, torch.int8, torch.float32, torch.int32,
                  {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2})
    return _TORCH


def _stream_ptr(stream, device: int | None = None):
    """Raw cudaStream_t of `stream`, or of the current stream of `device`."""
    torch = _torch()[0]
    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    if device is None:
        device = torch.cuda.current_device()
    return C.c_void_p(torch._C._cuda_getCurrentRawStream(device))


class Workspace:
    """lqg_workspace: a split-K scratch per concurrent stream."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(_lib.lib().lqg_workspace_create(device, C.byref(h)))
        self.handle, self.device = h, device

    def close(self):
        if self.handle:
            _lib.lib().lqg_workspace_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceWeights:
    """A device-resident, prepacked W4 weight handle (lqg_weights)."""

    def __init__(self, handle: C.c_void_p, device: int):
        self.handle, self.device = handle, device
        n, k, g = C.c_uint32(), C.c_uint32(), C.c_uint32()
        check(_lib.lib().lqg_weights_shape(handle, C.byref(n), C.byref(k), C.byref(g)))
        self.n, self.k, self.group_size = n.value, k.value, g.value

    @classmethod
    def from_bundle(cls, b: QuantizedWeightBundle, device: int = 0) -> "DeviceWeights":
        if b.group_scales.size != b.group_offsets.size:
            raise ValidationError("group parameter arrays have wrong size")
        v, _keep = b._view()
        h = C.c_void_p()
        check(_lib.lib().lqg_weights_create(C.byref(v), device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def from_image(cls, image: np.ndarray, channel_scales: np.ndarray, n: int, k: int,
                   group_size: int, device: int = 0) -> "DeviceWeights":
        """Upload a prepacked image (QuantizedWeightBundle.prepack / a cache file)."""
        img = np.ascontiguousarray(image, np.uint8)
        cs = np.ascontiguousarray(channel_scales, np.float32)
        if cs.size != n:
            raise ValidationError("channel scale array has wrong size")
        h = C.c_void_p()
        check(_lib.lib().lqg_weights_from_image(img.ctypes.data, img.size, cs.ctypes.data, n, k,
                                                group_size, device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def quantize(cls, w, group_size: int, stream=None) -> "DeviceWeights":
        """Two-level LiquidQuant of device FP32 weights [n, k] on the GPU
        (build_bundle, quant.cpp:203-232, bit-exact)."""
        import torch
        if not (w.is_cuda and w.dtype == torch.float32 and w.dim() == 2 and w.stride(1) == 1):
            raise ValidationError("weights must be a row-major CUDA float32 [n, k] tensor")
        h = C.c_void_p()
        check(_lib.lib().lqg_weights_quantize(w.data_ptr(), w.stride(0), w.shape[0], w.shape[1],
                                              group_size, _stream_ptr(stream), C.byref(h)))
        return cls(h, w.device.index)

    @classmethod
    def load(cls, path: str, device: int = 0) -> "DeviceWeights":
        """An LQWB bundle file (the reference's save_bundle format) straight to
        the device (lqg_weights_load: load_bundle's checks, device prepack)."""
        h = C.c_void_p()
        check(_lib.lib().lqg_weights_load(os.fsencode(path), device, C.byref(h)))
        return cls(h, device)

    def save(self, path: str) -> None:
        """Write this handle as a PlainRowMajor LQWB file (lqg_weights_save)."""
        check(_lib.lib().lqg_weights_save(self.handle, os.fsencode(path)))

    @property
    def device_bytes(self) -> int:
        return int(_lib.lib().lqg_weights_device_bytes(self.handle))

    def _check_x(self, xq):
        torch, i8 = _torch()[:2]
        if not (xq.dtype is i8 and xq.is_cuda and xq.dim() == 2 and xq.shape[1] == self.k
                and xq.stride(1) == 1):
            raise ValidationError(f"activations must be a CUDA int8 [m, {self.k}] row-major tensor")
        if xq.get_device() != self.device:
            raise ValidationError(f"activations live on cuda:{xq.get_device()}, weights on cuda:{self.device}")

    def _check_ts(self, ts, m):
        f32 = _torch()[2]
        if not (ts.dtype is f32 and ts.is_cuda and ts.dim() == 1 and ts.stride(0) == 1
                and ts.shape[0] >= m and ts.get_device() == self.device):
            raise ValidationError(f"token scales must be a contiguous CUDA float32 [>= {m}] tensor "
                                  f"on cuda:{self.device}")

    def _check_out(self, out, m, dtypes):
        if not (out.is_cuda and out.get_device() == self.device and out.dim() == 2
                and out.shape[0] == m and out.shape[1] == self.n and out.stride(1) == 1
                and out.stride(0) >= self.n):
            raise ValidationError(f"output must be a row-major CUDA [{m}, {self.n}] tensor on cuda:{self.device}")
        if str(out.dtype).replace("torch.", "") not in dtypes:
            raise ValidationError(f"unsupported output dtype {out.dtype}")

    def gemm(self, xq, ts, out=None, out_dtype=None, workspace: Workspace | None = None,
             stream=None):
        """Y[m, n] = (X_i8 @ W^_i8.T) * cs[n] * ts[m] in out_dtype (default bf16)."""
        torch, _, _, _, ycodes = _torch()
        self._check_x(xq)
        m = xq.shape[0]
        self._check_ts(ts, m)
        if out is None:
            out = torch.empty(m, self.n, dtype=out_dtype or torch.bfloat16, device=xq.device)
        elif not (out.is_cuda and out.get_device() == self.device and out.dim() == 2
                  and out.shape[0] == m and out.shape[1] == self.n and out.stride(1) == 1
                  and out.stride(0) >= self.n):
            raise ValidationError(f"output must be a row-major CUDA [{m}, {self.n}] tensor on cuda:{self.device}")
        code = ycodes.get(out.dtype)
        if code is None:
            raise ValidationError(f"unsupported output dtype {out.dtype}")
        check(_lib.lib().lqg_gemm_w4a8(
            self.handle, xq.data_ptr(), xq.stride(0), ts.data_ptr(), m, out.data_ptr(),
            out.stride(0), code, workspace.handle if workspace else None,
            _stream_ptr(stream, self.device)))
        return out

    def gemm_fanout(self, xq, ts, outs, workspace: Workspace | None = None, stream=None):
        """Y written by the epilogue into every tensor of `outs` (same shape and
        row pitch; local or peer-mapped device memory): lqg_gemm_w4a8_fanout.
        Each `out` may be a column slice of a wider row-major buffer."""
        self._check_x(xq)
        m = xq.shape[0]
        self._check_ts(ts, m)
        if not 1 <= len(outs) <= 8:
            raise ValidationError("1..8 output tensors")
        ld = outs[0].stride(0)
        for o in outs:
            if o.shape[0] < m or o.shape[1] != self.n or o.stride(0) != ld or o.stride(1) != 1 \
                    or o.dtype != outs[0].dtype or not o.is_cuda:
                raise ValidationError("fan-out outputs must share shape, dtype and row pitch")
        ptrs = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        check(_lib.lib().lqg_gemm_w4a8_fanout(
            self.handle, xq.data_ptr(), xq.stride(0), ts.data_ptr(), m, ptrs, len(outs), ld,
            _y_code(outs[0].dtype), workspace.handle if workspace else None, _stream_ptr(stream, self.device)))
        return outs[0]

    def gemm_accum(self, xq, out=None, workspace: Workspace | None = None, stream=None):
        import torch
        self._check_x(xq)
        m = xq.shape[0]
        if out is None:
            out = torch.empty(m, self.n, dtype=torch.int32, device=xq.device)
        self._check_out(out, m, ("int32",))
        check(_lib.lib().lqg_gemm_w4a8_accum(
            self.handle, xq.data_ptr(), xq.stride(0), m, out.data_ptr(), out.stride(0),
            workspace.handle if workspace else None, _stream_ptr(stream, self.device)))
        return out

    def gemm_host(self, x_host, ts_host, y_host, stream=None) -> None:
        """The reference-facing host-buffer call (lqg_gemm_w4a8_host): inputs
        and output live in host memory (pinned for full PCIe speed)."""
        import torch
        m = x_host.shape[0]
        check(_lib.lib().lqg_gemm_w4a8_host(self.handle, x_host.data_ptr(), ts_host.data_ptr(), m,
                                            y_host.data_ptr(), _y_code(y_host.dtype),
                                            _stream_ptr(stream, self.device)))

    def dequant(self, out=None, stream=None):
        """W^ as INT8 [n, k] through the mainloop's LQQ routine."""
        import torch
        if out is None:
            out = torch.empty(self.n, self.k, dtype=torch.int8, device=f"cuda:{self.device}")
        check(_lib.lib().lqg_dequant_weights(self.handle, out.data_ptr(), out.stride(0),
                                             _stream_ptr(stream, self.device)))
        return out

    def export(self) -> QuantizedWeightBundle:
        """Plain-layout host bundle of this handle."""
        n, k, g = self.n, self.k, self.group_size
        packed = np.zeros((n * k + 1) // 2, np.uint8)
        sc = np.zeros(n * (k // g), np.uint8)
        of = np.zeros(n * (k // g), np.uint8)
        cs = np.zeros(n, np.float32)
        check(_lib.lib().lqg_weights_export(self.handle, packed.ctypes.data, sc.ctypes.data,
                                            of.ctypes.data, cs.ctypes.data))
        return QuantizedWeightBundle(n, k, g, WeightLayout.PlainRowMajor, FragmentDescriptor(),
                                     packed, sc, of, cs)

    def close(self):
        if self.handle:
            _lib.lib().lqg_weights_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _group_args(weights, xq, m_list):
    import torch
    if len(weights) != len(m_list) or not weights:
        raise ValidationError("one token count per weight group is required")
    k = weights[0].k
    if not (xq.is_cuda and xq.dtype == torch.int8 and xq.dim() == 2 and xq.shape[1] == k
            and xq.stride(1) == 1):
        raise ValidationError(f"activations must be a CUDA int8 [rows, {k}] row-major tensor")
    ms = np.ascontiguousarray(m_list, np.uint32)
    if int(ms.sum()) != xq.shape[0]:
        raise ValidationError("sum of group token counts must equal the activation rows")
    handles = (C.c_void_p * len(weights))(*[w.handle for w in weights])
    return handles, ms


def gemm_grouped(weights, xq, ts, m_list, out=None, out_dtype=None,
                 workspace: Workspace | None = None, stream=None):
    """Grouped (MoE) W4A8 GEMM in one launch (lqg_gemm_w4a8_grouped): group e
    (weights[e], m_list[e] tokens) owns the next m_list[e] rows of xq / ts /
    out in order. Per group bit-identical to DeviceWeights.gemm."""
    import torch
    handles, ms = _group_args(weights, xq, m_list)
    if out is None:
        out = torch.empty(xq.shape[0], weights[0].n, dtype=out_dtype or torch.bfloat16,
                          device=xq.device)
    check(_lib.lib().lqg_gemm_w4a8_grouped(
        handles, len(weights), xq.data_ptr(), xq.stride(0), ts.data_ptr(), ms.ctypes.data,
        out.data_ptr(), out.stride(0), _y_code(out.dtype), workspace.handle if workspace else None,
        _stream_ptr(stream, xq.get_device())))
    return out


def gemm_grouped_accum(weights, xq, m_list, out=None, workspace: Workspace | None = None,
                       stream=None):
    """INT32 accumulators of the grouped GEMM."""
    import torch
    handles, ms = _group_args(weights, xq, m_list)
    if out is None:
        out = torch.empty(xq.shape[0], weights[0].n, dtype=torch.int32, device=xq.device)
    check(_lib.lib().lqg_gemm_w4a8_grouped_accum(
        handles, len(weights), xq.data_ptr(), xq.stride(0), ms.ctypes.data, out.data_ptr(),
        out.stride(0), workspace.handle if workspace else None, _stream_ptr(stream, xq.get_device())))
    return out


def quantize_activations(x, out_q=None, out_ts=None, check_finite: bool = False, stream=None):
    """Per-token INT8 quantization of a CUDA float32 [m, k] tensor
    (gemm.cpp:19-47, bit-exact). Returns (q int8 [m, k], ts float32 [m])."""
    import torch
    if not (x.is_cuda and x.dtype == torch.float32 and x.dim() == 2 and x.stride(1) == 1):
        raise ValidationError("activations must be a row-major CUDA float32 [m, k] tensor")
    m, k = x.shape
    q = out_q if out_q is not None else torch.empty(m, k, dtype=torch.int8, device=x.device)
    ts = out_ts if out_ts is not None else torch.empty(m, dtype=torch.float32, device=x.device)
    check(_lib.lib().lqg_quantize_activations(x.data_ptr(), x.stride(0), m, k, q.data_ptr(),
                                              q.stride(0), ts.data_ptr(), int(check_finite),
                                              _stream_ptr(stream, x.get_device())))
    return q, ts


def tune_set(name: str, value: int) -> None:
    """Set a launch-schedule knob (lqg_tune_set; results are bit-identical
    under every setting)."""
    check(_lib.lib().lqg_tune_set(name.encode(), int(value)))


def tune_get(name: str) -> int:
    v = C.c_int64()
    check(_lib.lib().lqg_tune_get(name.encode(), C.byref(v)))
    return v.value


class tune:
    """Context manager: ``with lq.tune(pair=1): ...`` sets knobs and restores
    their previous values on exit."""

    def __init__(self, **knobs):
        self.knobs = knobs
        self.old = {}

    def __enter__(self):
        for k, v in self.knobs.items():
            self.old[k] = tune_get(k)
            tune_set(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            tune_set(k, v)


def launch_count() -> int:
    """Kernels launched by liblqg.so in this process."""
    return int(_lib.lib().lqg_kernel_launch_count())
