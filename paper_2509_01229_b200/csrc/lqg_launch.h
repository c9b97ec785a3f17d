// Launch interface between the host API (lqg_api.cu) and the GEMM kernels.
// The kernels are instantiated per output kind in separate translation units
// (lqg_kern.cu compiled once per LQG_KIND), built in parallel; lqg_api.cu
// picks the unit by the call's output kind.
#pragma once
#include <cuda_runtime.h>

#include "lqg_gemm.cuh"

namespace lqg {

constexpr uint32_t kMaxGroups = 64;  // experts per grouped launch
constexpr uint32_t kSmemMax = 227 * 1024;

// Everything one GEMM launch needs, as plain values.
struct KernelSpec {
    CUtensorMap tmap_x;
    GemmParams p;
    const GroupTable<kMaxGroups>* gt;  // the groups (ng > 1: grouped kernel)
    uint32_t ng;
    bool pair, fan, pdl;
    uint32_t cluster;  // pair kernels: CTAs per cluster (2, or 4 in quad mode)
    uint32_t grid;
    size_t smem;
    cudaStream_t stream;
};

using LaunchFn = cudaError_t (*)(const KernelSpec&);
// Co-resident 2-CTA clusters of the pair kernel at this shared-memory size.
using PairClustersFn = int (*)(size_t smem, uint32_t grid);

#define LQG_DECLARE_KIND(K)                               \
    cudaError_t launch_gemm_kind##K(const KernelSpec& k); \
    int pair_clusters_kind##K(size_t smem, uint32_t grid, uint32_t cluster); \
    int debug_trace_kind##K(unsigned long long* out);
LQG_DECLARE_KIND(0)
LQG_DECLARE_KIND(1)
LQG_DECLARE_KIND(2)
LQG_DECLARE_KIND(3)
#undef LQG_DECLARE_KIND

}  // namespace lqg
