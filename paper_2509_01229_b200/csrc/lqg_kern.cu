// GEMM kernel instantiations for one output kind (LQG_KIND = OutKind), and
// their launch: plain, CTA-pair, fan-out, grouped and grouped-pair kernels.
#include "lqg_launch.h"

#ifndef LQG_KIND
#error "compile with -DLQG_KIND=<0..3> (lqg::OutKind)"
#endif
#define LQG_CAT2(a, b) a##b
#define LQG_CAT(a, b) LQG_CAT2(a, b)

namespace lqg {
namespace {

template <uint32_t kG, bool kFan, bool kPair>
cudaError_t smem_attr() {
    static const cudaError_t e = cudaFuncSetAttribute(lqg_w4a8_gemm_kernel<LQG_KIND, kG, kFan, kPair>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
    return e;
}

template <uint32_t kG, bool kFan, bool kPair, typename GT>
cudaError_t launch(const KernelSpec& k, const GT& gt) {
    cudaError_t e = smem_attr<kG, kFan, kPair>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(k.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = k.smem;
    cfg.stream = k.stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = k.pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = kPair ? k.cluster : 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = kPair ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, lqg_w4a8_gemm_kernel<LQG_KIND, kG, kFan, kPair>, k.tmap_x, k.p, gt);
}

}  // namespace

cudaError_t LQG_CAT(launch_gemm_kind, LQG_KIND)(const KernelSpec& k) {
    if (k.ng > 1) return k.pair ? launch<kMaxGroups, false, true>(k, *k.gt) : launch<kMaxGroups, false, false>(k, *k.gt);
    GroupTable<1> g1{};
    g1.e[0] = k.gt->e[0];
    g1.n = 1;
    if (k.pair) return launch<1, false, true>(k, g1);
    if (k.fan) return launch<1, true, false>(k, g1);
    return launch<1, false, false>(k, g1);
}

int LQG_CAT(pair_clusters_kind, LQG_KIND)(size_t smem, uint32_t grid, uint32_t cluster) {
    if (smem_attr<1, false, true>() != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, lqg_w4a8_gemm_kernel<LQG_KIND, 1, false, true>, &cfg) != cudaSuccess)
        nc = 0;
    cudaGetLastError();
    return nc;
}

#ifdef LQG_TRACE_KB
// LQG_TRACE_KB builds: this unit's per-k-block event buffer of CTA 0.
extern "C" int LQG_CAT(lqg_debug_kb_kind, LQG_KIND)(long long* out) {
    return cudaMemcpyFromSymbol(out, g_lqg_kb, sizeof(long long) * 2 * 64 * 8) == cudaSuccess ? 0 : 4;
}
#endif

#ifdef LQG_TRACE_SEG
// LQG_TRACE_SEG builds: this unit's per-segment event buffer of CTAs 0..7.
extern "C" int LQG_CAT(lqg_debug_seg_kind, LQG_KIND)(long long* out) {
    return cudaMemcpyFromSymbol(out, g_lqg_seg, sizeof(long long) * 8 * 32 * 16) == cudaSuccess ? 0 : 4;
}
#endif

// LQG_TRACE builds: this unit's per-CTA event buffer (zeros otherwise).
int LQG_CAT(debug_trace_kind, LQG_KIND)(unsigned long long* out) {
#ifdef LQG_TRACE
    return cudaMemcpyFromSymbol(out, g_lqg_trace, sizeof(unsigned long long) * 8 * 160 * 16) == cudaSuccess ? 0 : 4;
#else
    for (size_t i = 0; i < size_t(8) * 160 * 16; ++i) out[i] = 0;
    return 0;
#endif
}

}  // namespace lqg
