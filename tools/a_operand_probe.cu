// Where should the dequantized INT8 A operand live: TMEM (the product:
// tcgen05.st by the dequant warps, tcgen05.mma ... [a_tmem]) or swizzled
// shared memory (STS.128 into the SW128 K-major layout + fence.proxy.async,
// tcgen05.mma with an A descriptor)? Per 256-wide k-block of a 128-row
// weight tile this probe times, on every SM at once:
//   * the MMA warp alone: 8 x tcgen05.mma.kind::i8 (K = 32 each) + commit,
//     A from TMEM vs A from SMEM, N = 16 / 128 / 192 / 256;
//   * one dequant warpgroup alone writing a k-block (thread = row, 256 B):
//     2 x tcgen05.st.32x32b.x32 + wait::st vs 16 x STS.128 + proxy fence;
//   * both at once (two A slots: the writers fill one while the MMAs read the
//     other), i.e. with the shared-memory traffic of both paths competing.
// Operand contents are irrelevant (timing only); there is no hand-off between
// the roles, each runs its own loop.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2509_01229_b200/csrc tools/a_operand_probe.cu -o tools/a_probe.bin
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_ptx.cuh"

using namespace lqg;

namespace {

__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

constexpr uint32_t kASlot = 128 * 256;  // one k-block of A: 128 rows x 256 int8
constexpr uint32_t kBBytes = 256 * 256; // B: up to 256 tokens x 256 int8
constexpr uint32_t kSmem = 2 * kASlot + kBBytes + 1024;

// kMode bit 0: run the MMA warp, bit 1: run the writer warpgroup.
template <bool kSmemA, int kMode>
__global__ void __launch_bounds__(256, 1) probe(uint32_t n_dim, uint32_t iters, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t holder;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&holder), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t a_smem = ptx::smem_u32(smem), b_smem = a_smem + 2 * kASlot;
    if (warp == 0 && (kMode & 1)) {
        const uint32_t idesc = ptx::idesc_i8(128, n_dim);
        const uint64_t bdesc = ptx::sw128_kmajor_desc(b_smem);
        const uint32_t b0 = ptx::smem_u32(&bar);
        __syncwarp();
        const long long t0 = clock64();
        for (uint32_t it = 0; it < iters; ++it) {
            if (ptx::elect_one()) {
                const uint32_t slot = it & 1;
                for (uint32_t k = 0; k < 8; ++k) {
                    // K-major SW128: 32-byte k steps inside a 128-byte atom
                    // (+2 in 16-byte descriptor units), the second atom column
                    // 16 KB further (128 rows x 128 B)
                    const uint64_t koff = (k % 4) * 2 + (k / 4) * (16384 >> 4);
                    if (kSmemA)
                        mma_i8_ss(tmem,
                                  ptx::sw128_kmajor_desc(a_smem + slot * kASlot) + koff,
                                  bdesc + (k % 4) * 2, idesc, k ? 1u : 0u);
                    else
                        ptx::mma_i8_ts(tmem, tmem + 384 + slot * 64 + k * 8,
                                       bdesc + (k % 4) * 2, idesc, k ? 1u : 0u);
                }
                ptx::mma_commit(b0);
            }
            __syncwarp();
        }
        // wait for the last commit: every issued MMA has completed
        ptx::mbar_wait(b0, (iters - 1) & 1);
        const long long t1 = clock64();
        if (threadIdx.x == 0) out[2 * blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    if (warp >= 4 && (kMode & 2)) {
        const uint32_t row = (warp % 4) * 32 + lane;
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = row * 131 + i;
        const long long t0 = clock64();
        for (uint32_t it = 0; it < iters; ++it) {
            const uint32_t slot = (it & 1) ^ 1;  // the slot the MMAs are not reading
            if (kSmemA) {
                // row r, 16-byte chunk c of atom column a: byte offset
                // a * 16384 + (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) * 16)
                const uint32_t base = a_smem + slot * kASlot + (row / 8) * 1024 + (row % 8) * 128;
#pragma unroll
                for (uint32_t c = 0; c < 16; ++c) {
                    const uint32_t addr = base + (c / 8) * 16384 + (((c % 8) ^ (row % 8)) * 16);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v[(2 * c) % 32] + it),
                                 "r"(v[(2 * c + 1) % 32]), "r"(v[(2 * c + 2) % 32]), "r"(v[(2 * c + 3) % 32])
                                 : "memory");
                }
                ptx::fence_proxy_async();
            } else {
                const uint32_t taddr = tmem + ((warp % 4) * 32 << 16) + 384 + slot * 64;
                v[0] += it;
                ptx::tmem_st_x32(taddr, v);
                ptx::tmem_st_x32(taddr + 32, v);
                ptx::tmem_st_wait();
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");  // the warpgroup publishes the slot together
        }
        const long long t1 = clock64();
        if (threadIdx.x == 128) out[2 * blockIdx.x + 1] = (unsigned long long)(t1 - t0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16 * 148);
    cudaMemset(d, 0, 16 * 148);
    auto run = [&](auto kern, const char* name, uint32_t n) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        const uint32_t iters = 4000;
        kern<<<148, 256, kSmem>>>(n, iters, d);
        kern<<<148, 256, kSmem>>>(n, iters, d);
        const cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[2 * 148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mma = 0, wr = 0;
        for (int i = 0; i < 148; ++i) {
            mma += h[2 * i];
            wr += h[2 * i + 1];
        }
        mma /= 148.0 * iters;
        wr /= 148.0 * iters;
        printf("%-34s N=%3u: MMA %7.1f cyc/k-block (floor %5.0f)  writer %7.1f cyc/k-block  %s\n", name, n, mma,
               4.0 * n, wr, cudaGetErrorString(e));
        cudaMemset(d, 0, 16 * 148);
    };
    for (uint32_t n : {16u, 128u, 192u, 256u}) {
        run(probe<false, 1>, "A in TMEM:  MMA only", n);
        run(probe<true, 1>, "A in SMEM:  MMA only", n);
        run(probe<false, 3>, "A in TMEM:  MMA + writer", n);
        run(probe<true, 3>, "A in SMEM:  MMA + writer", n);
    }
    run(probe<false, 2>, "A in TMEM:  writer only", 128);
    run(probe<true, 2>, "A in SMEM:  writer only", 128);
    return 0;
}
