"""ctypes binding of liblqg.so (include/lqg.h) and its in-tree build.

The library is built in-tree (``paper_2509_01229_b200/liblqg.so``) with nvcc
for sm_100a only. There is no CPU fallback: if the library is missing the
import of the compute entry points fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("LQG_LIB_PATH") or os.path.join(HERE, "liblqg.so")
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["lqg_api.cu", "lqg_kern.cu"]
HEADERS = ["lqg_gemm.cuh", "lqg_aux.cuh", "lqg_layout.h", "sm100_ptx.cuh", "lqg_launch.h"]
# lqg_kern.cu is compiled once per output kind (lqg::OutKind 0..3), in parallel
KINDS = (0, 1, 2, 3)

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC",
]


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "lqg.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: str | None = None) -> str:
    """Compile liblqg.so for sm_100a (cross-compiles without a GPU): the host
    API and the four per-output-kind kernel units are compiled in parallel,
    then linked. `defines` and `out` build debug variants (e.g. -DLQG_TRACE
    into liblqg_trace.so)."""
    import shutil
    import tempfile
    target = out or LIB_PATH
    if not force and not out and not _stale():
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    base = [nvcc, *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines]]
    tmp = tempfile.mkdtemp(prefix="lqg_build_")
    try:
        units = [(os.path.join(CSRC, "lqg_api.cu"), os.path.join(tmp, "api.o"), [])]
        units += [(os.path.join(CSRC, "lqg_kern.cu"), os.path.join(tmp, f"kern{k}.o"), [f"-DLQG_KIND={k}"])
                  for k in KINDS]
        procs = [subprocess.Popen([*base, *extra, "-c", "-o", obj, src]) for src, obj, extra in units]
        rcs = [pr.wait() for pr in procs]
        if any(rcs):
            raise subprocess.CalledProcessError(max(rcs), "nvcc")
        subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", target + ".tmp",
                        *[obj for _, obj, _ in units]], check=True)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    os.replace(target + ".tmp", target)
    return target


class FragmentDescriptorC(C.Structure):
    _fields_ = [("warps_per_group", C.c_uint8), ("threads_per_warp", C.c_uint8),
                ("mma_m", C.c_uint16), ("mma_k", C.c_uint16),
                ("elements_per_thread_per_mma", C.c_uint16), ("dual_k_span", C.c_uint16)]


class BundleViewC(C.Structure):
    _fields_ = [("n", C.c_uint32), ("k", C.c_uint32), ("group_size", C.c_uint32),
                ("layout", C.c_uint32), ("fragment", FragmentDescriptorC),
                ("packed_weights", C.c_void_p), ("packed_bytes", C.c_uint64),
                ("group_scales", C.c_void_p), ("group_offsets", C.c_void_p),
                ("n_groups", C.c_uint64), ("channel_scales", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load liblqg.so (building it first if it is missing or stale and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if (not os.environ.get("LQG_LIB_PATH") and _stale()
            and os.path.exists(os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"))):
        build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, u32, i32 = C.c_void_p, C.c_int64, C.c_uint32, C.c_int
    sig = {
        "lqg_bundle_validate": [C.POINTER(BundleViewC)],
        "lqg_weights_create": [C.POINTER(BundleViewC), i32, C.POINTER(vp)],
        "lqg_prepack_host": [C.POINTER(BundleViewC), vp, C.c_uint64],
        "lqg_weights_from_image": [vp, C.c_uint64, vp, u32, u32, u32, i32, C.POINTER(vp)],
        "lqg_weights_quantize": [vp, i64, u32, u32, u32, vp, C.POINTER(vp)],
        "lqg_weights_destroy": [vp],
        "lqg_weights_load": [C.c_char_p, i32, C.POINTER(vp)],
        "lqg_bundle_file_validate": [C.c_char_p],
        "lqg_weights_save": [vp, C.c_char_p],
        "lqg_weights_shape": [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)],
        "lqg_weights_export": [vp, vp, vp, vp, vp],
        "lqg_workspace_create": [i32, C.POINTER(vp)],
        "lqg_workspace_destroy": [vp],
        "lqg_gemm_w4a8": [vp, vp, i64, vp, u32, vp, i64, i32, vp, vp],
        "lqg_gemm_w4a8_accum": [vp, vp, i64, u32, vp, i64, vp, vp],
        "lqg_gemm_w4a8_fanout": [vp, vp, i64, vp, u32, vp, u32, i64, i32, vp, vp],
        "lqg_gemm_w4a8_grouped": [vp, u32, vp, i64, vp, vp, vp, i64, i32, vp, vp],
        "lqg_gemm_w4a8_grouped_accum": [vp, u32, vp, i64, vp, vp, i64, vp, vp],
        "lqg_gemm_w4a8_host": [vp, vp, vp, u32, vp, i32, vp],
        "lqg_gemm_w4a8_accum_host": [vp, vp, u32, vp, vp],
        "lqg_dequant_weights": [vp, vp, i64, vp],
        "lqg_quantize_activations": [vp, i64, u32, u32, vp, i64, vp, i32, vp],
    }
    for name, args in sig.items():
        # an older build (A/B timing via LQG_LIB_PATH) may lack newer entry
        # points; tests/test_boundary.py checks the in-tree library exports all
        f = getattr(L, name, None)
        if f is None:
            continue
        f.argtypes = args
        f.restype = C.c_int
    if hasattr(L, "lqg_tune_set"):
        L.lqg_tune_set.argtypes = [C.c_char_p, i64]
        L.lqg_tune_set.restype = C.c_int
        L.lqg_tune_get.argtypes = [C.c_char_p, C.POINTER(i64)]
        L.lqg_tune_get.restype = C.c_int
        L.lqg_tune_reset.restype = None
    L.lqg_image_bytes.argtypes = [u32, u32, u32]
    L.lqg_image_bytes.restype = C.c_uint64
    L.lqg_weights_device_bytes.argtypes = [vp]
    L.lqg_weights_device_bytes.restype = C.c_uint64
    L.lqg_kernel_launch_count.restype = C.c_uint64
    L.lqg_last_error.restype = C.c_char_p
    L.lqg_version.restype = C.c_char_p
    _lib = L
    return L


# Symbols declared in include/lqg.h (checked by tests/test_boundary.py).
EXPORTS = [
    "lqg_bundle_validate", "lqg_image_bytes", "lqg_prepack_host", "lqg_weights_from_image",
    "lqg_weights_create", "lqg_weights_quantize", "lqg_weights_destroy",
    "lqg_weights_load", "lqg_bundle_file_validate", "lqg_weights_save",
    "lqg_weights_shape", "lqg_weights_export", "lqg_weights_device_bytes",
    "lqg_workspace_create", "lqg_workspace_destroy", "lqg_gemm_w4a8", "lqg_gemm_w4a8_accum",
    "lqg_gemm_w4a8_grouped", "lqg_gemm_w4a8_grouped_accum", "lqg_gemm_w4a8_fanout",
    "lqg_gemm_w4a8_host", "lqg_gemm_w4a8_accum_host", "lqg_dequant_weights",
    "lqg_quantize_activations", "lqg_kernel_launch_count", "lqg_tune_set", "lqg_tune_get",
    "lqg_tune_reset", "lqg_last_error", "lqg_version",
]
