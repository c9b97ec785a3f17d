// Cost structure of the MMA-issuer loop on sm_100a: cycles per iteration of
// tcgen05.mma.kind::i8 (A in TMEM, B from a SW128 shared-memory descriptor)
// issue, with and without commits, satisfied mbarrier waits and fences, for
// N = 16 / 128 / 256 (M = 128, K = 32 per MMA). Operand contents are
// irrelevant (timing only).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2509_01229_b200/csrc tools/mma_issue_probe.cu -o tools/mma_probe.bin
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_ptx.cuh"

using namespace lqg;

template <int kVariant>
__global__ void __launch_bounds__(128, 1) probe(uint32_t n_dim, uint32_t iters, uint32_t mmas, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t holder;
    __shared__ __align__(8) uint64_t bars[4];
    const uint32_t warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) ptx::mbar_init(ptx::smem_u32(&bars[i]), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&holder), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = holder;
    if (warp == 0) {
        const uint32_t idesc = ptx::idesc_i8(128, n_dim);
        const uint64_t desc = ptx::sw128_kmajor_desc(ptx::smem_u32(smem));
        const uint32_t b0 = ptx::smem_u32(&bars[0]);
        // bars[3] is never arrived on: parity 1 reads as complete
        const uint32_t done = ptx::smem_u32(&bars[3]);
        __syncwarp();
        const long long t0 = clock64();
        for (uint32_t it = 0; it < iters; ++it) {
            if (kVariant >= 2) ptx::mbar_wait(done, 1);
            if (kVariant >= 3) ptx::tc_fence_after();
            if (ptx::elect_one()) {
                for (uint32_t k = 0; k < mmas; ++k)
                    ptx::mma_i8_ts(tmem + (it & 1) * 256, tmem + 384 + k * 8, desc + (k % 4) * 2, idesc, k ? 1u : 0u);
                if (kVariant >= 1) {
                    ptx::mma_commit(b0);
                    ptx::mma_commit(b0 + 8);
                }
            }
            __syncwarp();
        }
        const long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8 * 148);
    auto run = [&](auto kern, const char* name, uint32_t n, uint32_t mmas) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        const uint32_t iters = 2000;
        kern<<<148, 128, 64 * 1024>>>(n, iters, mmas, d);
        kern<<<148, 128, 64 * 1024>>>(n, iters, mmas, d);
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148.0 * iters;
        const double floor = 128.0 * n / 256.0 * mmas;
        printf("%-28s N=%3u mmas=%2u: %7.1f cyc/iter  (MMA floor %6.1f)  %s\n", name, n, mmas, avg, floor,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (uint32_t n : {16u, 128u, 256u}) {
        run(probe<0>, "mma only", n, 8);
        run(probe<1>, "mma + 2 commits", n, 8);
        run(probe<2>, "+ satisfied wait", n, 8);
        run(probe<3>, "+ fence", n, 8);
        run(probe<3>, "+ fence, 16 mma", n, 16);
        run(probe<3>, "+ fence, 4 mma", n, 4);
    }
    return 0;
}
