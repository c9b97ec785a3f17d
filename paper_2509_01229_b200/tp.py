"""Column-sharded (N-split) W4A8 linear across the ranks of a process group.

North star, subsystem 4: LLaMA-class layer weights are split by output
channel across 1/2/4/8 GPUs of one node; activations (INT8 codes + per-token
scales) are replicated, each rank computes its column slice with the sm_100a
kernel, and the row output is all-gathered with NCCL over NVLink. Integer
accumulators and the per-element epilogue are shard-invariant, so the gathered
Y equals the single-GPU Y byte for byte.

Rank r owns weight rows [start_r, end_r), 128-row aligned (one tcgen05 M tile)
so every shard is a whole number of device tiles; shards are padded to the
largest one for the fixed-size all-gather.

Two gather modes:
  * "nccl" (default): the kernel writes Y_r, then one NCCL all_gather_into_tensor
    over NVLink plus a strided copy (`gather_columns`).
  * "p2p": the row output lives in NVLink symmetric memory
    (torch.distributed._symmetric_memory); every rank's GEMM epilogue stores
    its column slice straight into every rank's Y (lqg_gemm_w4a8_fanout), so
    the all-gather is fused into the GEMM tile by tile and only a cross-GPU
    barrier remains.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .lq import QuantizedWeightBundle, ValidationError, WeightLayout

TILE = 128


def shard_rows(n: int, world: int, align: int = TILE) -> list[tuple[int, int]]:
    """Contiguous, `align`-aligned row ranges covering [0, n), as even as possible."""
    if world < 1:
        raise ValidationError("world size must be >= 1")
    units = -(-n // align)
    out = []
    for r in range(world):
        u0, u1 = units * r // world, units * (r + 1) // world
        out.append((min(n, u0 * align), min(n, u1 * align)))
    return out


def slice_bundle(b: QuantizedWeightBundle, r0: int, r1: int) -> QuantizedWeightBundle:
    """Rows [r0, r1) of a bundle, in either reference layout (bundle.hpp:5-24):
    plain payload rows are k/2 bytes each (k is even for any device-supported
    group size); dual-MMA payload is 64-row bands of k/2*64 bytes."""
    n, k, g = b.n, b.k, b.group_size
    if not (0 <= r0 < r1 <= n):
        raise ValidationError("bad row range")
    gpr = k // g
    if b.layout == WeightLayout.PlainRowMajor:
        if k % 2:
            raise ValidationError("row slicing of a plain bundle needs an even k")
        packed = b.packed_weights[r0 * k // 2:r1 * k // 2]
    else:
        band = b.fragment.mma_m
        if r0 % band or (r1 % band and r1 != n):
            raise ValidationError(f"dual-MMA shards must be {band}-row aligned")
        packed = b.packed_weights[r0 * k // 2:r1 * k // 2]
    return QuantizedWeightBundle(r1 - r0, k, g, b.layout, b.fragment, np.ascontiguousarray(packed),
                                 np.ascontiguousarray(b.group_scales[r0 * gpr:r1 * gpr]),
                                 np.ascontiguousarray(b.group_offsets[r0 * gpr:r1 * gpr]),
                                 np.ascontiguousarray(b.channel_scales[r0:r1]))


@dataclass
class ShardPlan:
    n: int
    world: int
    rank: int
    ranges: list

    @property
    def rows(self) -> tuple[int, int]:
        return self.ranges[self.rank]

    @property
    def width(self) -> int:
        return max(e - s for s, e in self.ranges)


def gather_columns(y_local, plan: ShardPlan, group=None, out=None, buf=None):
    """All-gather the per-rank column slices [m, n_r] into Y [m, n] (row-major).

    One fixed-size all_gather_into_tensor of [world, m, width] (shards padded to
    the widest), then a strided copy into Y. Works with NCCL (GPU) and gloo (CPU).
    Allocation-free when the caller passes y_local already padded to the shard
    width (the GEMM can write straight into it: its output pitch is free), a
    gather buffer `buf` of >= world*m*width elements and `out` -- which is how
    the bench captures the N-split step in a CUDA graph.
    """
    import torch
    import torch.distributed as dist
    m = y_local.shape[0]
    s, e = plan.rows
    w = plan.width
    send = y_local
    if y_local.shape[1] != w or not y_local.is_contiguous():
        send = torch.zeros(m, w, dtype=y_local.dtype, device=y_local.device)
        send[:, :e - s] = y_local[:, :e - s]
    if buf is None:
        buf = torch.empty(plan.world * m * w, dtype=y_local.dtype, device=y_local.device)
    buf = buf[:plan.world * m * w]
    if plan.world > 1:
        dist.all_gather_into_tensor(buf, send.reshape(-1), group=group)
    else:
        buf.copy_(send.reshape(-1))
    parts = buf.view(plan.world, m, w)
    if out is None:
        out = torch.empty(m, plan.n, dtype=y_local.dtype, device=y_local.device)
    if all(e - s == w for s, e in plan.ranges) and plan.n == w * plan.world:
        out.view(m, plan.world, w).copy_(parts.transpose(0, 1))
    else:
        for r, (rs, re) in enumerate(plan.ranges):
            out[:, rs:re] = parts[r, :, :re - rs]
    return out


class ColumnParallelW4A8:
    """One W4A8 linear layer split by output channel across a process group.

    `local_gemm(xq, ts) -> Y_r [m, n_r]` defaults to the sm_100a kernel of this
    rank's DeviceWeights; tests on CPU inject a reference implementation to
    exercise the sharding and collective logic with gloo.
    """

    def __init__(self, n: int, k: int, group_size: int, rank: int, world: int, group=None,
                 local_gemm: Callable | None = None, device_weights=None, gather: str = "nccl"):
        if gather not in ("nccl", "p2p"):
            raise ValidationError("gather must be 'nccl' or 'p2p'")
        self.n, self.k, self.group_size = n, k, group_size
        self.plan = ShardPlan(n, world, rank, shard_rows(n, world))
        self.group = group
        self.dw = device_weights
        self._local = local_gemm
        self.gather = gather
        self._symm = None  # {"max_m", "dtype", "bufs": 2 x (local Y, every rank's Y, handle), "barrier"}
        self._symm_injected = False
        self._fanout = None
        self._calls = 0

    @classmethod
    def from_bundle(cls, b: QuantizedWeightBundle, rank: int, world: int, group=None,
                    device: int | None = None, local_gemm: Callable | None = None):
        """Each rank prepacks and uploads only its own rows of the full bundle."""
        self = cls(b.n, b.k, b.group_size, rank, world, group, local_gemm)
        s, e = self.plan.rows
        self.shard = slice_bundle(b, s, e)
        if local_gemm is None:
            from .lq import DeviceWeights
            self.dw = DeviceWeights.from_bundle(self.shard, device if device is not None else 0)
        return self

    @classmethod
    def from_weights(cls, w_full, group_size: int, rank: int, world: int, group=None):
        """Quantize this rank's rows of device FP32 weights [n, k] on its GPU."""
        from .lq import DeviceWeights
        n, k = w_full.shape
        self = cls(n, k, group_size, rank, world, group)
        s, e = self.plan.rows
        self.dw = DeviceWeights.quantize(w_full[s:e].contiguous(), group_size)
        return self

    def local(self, xq, ts, out=None):
        if self._local is not None:
            return self._local(xq, ts)
        return self.dw.gemm(xq, ts, out=out)

    def _symmetric_output(self, m: int, dtype, device):
        """Two Y buffers [max_m, n] in NVLink symmetric memory on every rank
        (double-buffered across calls) + every rank's view of them."""
        import torch.distributed as dist
        if self._symm is not None and self._symm["max_m"] >= m and self._symm["dtype"] == dtype:
            return self._symm
        import torch.distributed._symmetric_memory as symm_mem
        max_m = max(m, self._symm["max_m"] if self._symm else 0)
        world = self.plan.world
        bufs = []
        hdl = None
        for _ in range(2):
            y = symm_mem.empty(max_m, self.n, dtype=dtype, device=device)
            if world > 1:
                group = self.group if self.group is not None else dist.group.WORLD
                hdl = symm_mem.rendezvous(y, group)
                peers = [y if r == self.plan.rank else hdl.get_buffer(r, [max_m, self.n], dtype)
                         for r in range(world)]
            else:
                peers = [y]
            bufs.append((y, peers, hdl))
        self._symm = {"max_m": max_m, "dtype": dtype, "bufs": bufs,
                      "barrier": (lambda h=hdl: h.barrier()) if hdl is not None else (lambda: None)}
        return self._symm

    def forward(self, xq, ts, out=None, y_local=None, out_dtype=None):
        """Y [m, n] = gather_r( X W_r^T * cs_r * ts ), returned in `out` (or a
        new tensor) -- never a view of the shared gather buffers.

        p2p protocol (fused all-gather): call t's fan-out GEMM stores this
        rank's column slice into buffer t % 2 of every rank, then a cross-GPU
        barrier, then each rank copies its own buffer out. Call t + 2 writes
        the same buffer again only after the barrier of call t + 1, which no
        rank passes before every rank has finished its copy-out of call t
        (stream order: copy-out t, fan-out t+1, barrier t+1): no
        write-after-read race between a fast and a slow rank.
        """
        if self.gather == "p2p":
            import torch
            m = xq.shape[0]
            dtype = out_dtype or (out.dtype if out is not None else torch.bfloat16)
            symm = self._symm if self._symm_injected else self._symmetric_output(m, dtype, xq.device)
            y, peers, _ = symm["bufs"][self._calls % 2]
            self._calls += 1
            s, e = self.plan.rows
            # this rank's column slice of every rank's Y (itself first)
            me = self.plan.rank
            order = [me] + [r for r in range(self.plan.world) if r != me]
            dests = [peers[r][:m, s:e] for r in order]
            if self._fanout is not None:
                self._fanout(xq, ts, dests)
            else:
                self.dw.gemm_fanout(xq, ts, dests)
            symm["barrier"]()  # every rank's slices of call t have landed in every Y
            if out is None:
                out = torch.empty(m, self.n, dtype=dtype, device=xq.device)
            out.copy_(y[:m])
            return out
        y_r = self.local(xq, ts, out=y_local)
        return gather_columns(y_r, self.plan, self.group, out=out)

    def inject_symmetric(self, bufs, barrier, fanout):
        """Testing hook: run the p2p protocol over caller-provided buffers
        (bufs[slot] = (local Y, [Y of every rank])), barrier and fan-out
        function (e.g. process-shared CPU tensors and a gloo barrier)."""
        self._symm = {"max_m": bufs[0][0].shape[0], "dtype": bufs[0][0].dtype,
                      "bufs": [(b[0], b[1], None) for b in bufs], "barrier": barrier}
        self._symm_injected = True
        self._fanout = fanout
        self.gather = "p2p"

    __call__ = forward
