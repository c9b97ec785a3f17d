"""paper_2509_01229_b200 — a B200-native (sm_100a) LiquidGEMM W4A8 GEMM.

The hot path of arXiv 2509.01229 (LiquidGEMM): packed UINT4 weights with
LiquidQuant two-level scales, INT8 activations with per-token scales,
F32/F16/BF16 output — hand-written tcgen05/TMEM/TMA CUDA in liblqg.so behind
the C ABI of include/lqg.h, with a host-side mirror of the reference's
``namespace lq`` interface (``lq`` submodule) and a torch-level device API.

There is no CPU fallback: compute entry points raise if liblqg.so is missing
or no sm_100 device is present.
"""
from . import _lib
from .lq import (ActivationQuant, CudaError, DeviceWeights, Engine, FragmentDescriptor, GemmShape,
                 IoError, QuantizedWeightBundle, TileConfig, UnsupportedDeviceError,
                 ValidationError, VerificationError, WeightLayout, Workspace, gemm_grouped,
                 gemm_grouped_accum, gemm_w4a8, gemm_w4a8_accum, launch_count, quantize_activations,
                 quantize_activations_per_token, tune, tune_get, tune_set)

__all__ = [
    "ActivationQuant", "CudaError", "DeviceWeights", "Engine", "FragmentDescriptor", "GemmShape",
    "IoError", "QuantizedWeightBundle", "TileConfig", "UnsupportedDeviceError", "ValidationError",
    "VerificationError", "WeightLayout", "Workspace", "gemm_grouped", "gemm_grouped_accum",
    "gemm_w4a8", "gemm_w4a8_accum",
    "launch_count", "quantize_activations", "quantize_activations_per_token", "tune", "tune_get",
    "tune_set", "build",
]


def build(force: bool = False) -> str:
    """Compile liblqg.so for sm_100a in-tree."""
    return _lib.build(force=force)
