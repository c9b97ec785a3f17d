// The LiquidGEMM W4A8 mainloop for sm_100a (B200).
//
// Reference semantics: lq::gemm_w4a8_accum / lq::gemm_w4a8
// (/root/reference/proj/src/gemm.cpp:138-223): exact INT32 accumulation of
// x_i8 * w^_i8 over k, w^ = LQQ-dequantized UINT4 (packed.cpp:63-71), then
// y = float(double(acc) * double(cs[n]) * double(ts[m])) (quant.cpp:125-127).
//
// Hardware mapping (swap-AB: the tcgen05 M dimension is the weight row):
//   D[128 rows x BN tokens] (INT32, TMEM) += A[128 x 32] (int8, TMEM) * B[32 x BN] (int8, SMEM)
//
// Warp roles in one 512-thread CTA (one CTA per SM, persistent, stream-K):
//   warp 0        TMA producer: per k-block, one 1-D bulk copy of the
//                 prepacked weight chunk (codes + group params, EVICT_FIRST)
//                 and one 2-D SW128 tensor copy of the activation tile
//                 (EVICT_LAST) into an S-stage shared-memory ring.
//   warp 1        MMA issuer: 4 x tcgen05.mma.kind::i8 (K=32 each) per
//                 k-block, A read from TMEM, B from the swizzled ring slot;
//                 tcgen05.commit frees the ring slot / the TMEM A slot and
//                 signals the epilogue at the end of a tile segment.
//   warp 2        TMEM allocator (512 columns).
//   warps 4-11    two dequant warpgroups (ImFP) taking alternate
//                 k-blocks: LDS.128 of packed codes, LiquidQuant
//                 (q*s + a) ^ 0x80 on four byte lanes per IMAD
//                 (packed.cpp:40-61), tcgen05.st of the INT8
//                 result into the TMEM A ring (thread = weight row = lane).
//   warps 12-15   epilogue: tcgen05.ld of the INT32 accumulators, fused
//                 per-channel x per-token scaling and F32/F16/BF16 cast,
//                 coalesced stores (or the INT32 accumulators themselves).
// All hand-offs are mbarrier arrivals (TMA complete_tx, tcgen05.commit,
// thread arrives); there is no __syncthreads in the mainloop.
//
// Stream-K: the linear space of (tile, k-block) iterations is cut into
// gridDim.x contiguous ranges. A tile whose k-range is split between CTAs is
// reduced exactly in INT32 (red.global.add into a per-launch workspace slot,
// then the CTA that completes the tile's k-count applies the epilogue and
// re-zeroes the slot). Integer addition is associative, so the result is
// bit-identical to the reference's fixed-order sum.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "lqg_layout.h"
#include "sm100_ptx.cuh"

namespace lqg {

enum OutKind : uint32_t { kOutAcc = 0, kOutF32 = 1, kOutF16 = 2, kOutBF16 = 3 };

constexpr uint32_t kThreads = 512;
constexpr uint32_t kMaxStages = 16;
constexpr uint32_t kAStages = 8;           // TMEM A ring: 8 x 32 columns
constexpr uint32_t kAColBase = 256;        // A ring lives in TMEM columns [256, 512)
constexpr uint32_t kTmemCols = 512;

struct GemmParams {
    const uint8_t* wimg;       // prepacked weight image
    const float* cs;           // channel scales (padded to NT*128)
    const float* ts;           // token scales (m)
    void* out;                 // y or acc
    int64_t ldo;               // row pitch of out, in elements
    int32_t* ws;               // split-K workspace: gridDim.x slots of BN*128 int32
    uint32_t* counters;        // gridDim.x k-block counters
    uint32_t M, N;             // logical problem (tokens, weight rows)
    uint32_t KB, NT, MT;       // k-blocks, weight tiles, token tiles
    uint32_t BN;               // tokens per tile (16..256, multiple of 16)
    uint32_t P;                // group params per k-block (1, 2, 4)
    uint32_t chunk_bytes;      // bytes per (tile, k-block) weight chunk
    uint32_t stages;           // shared-memory ring depth
    uint32_t stage_bytes;      // bytes per ring slot (X tile first, then W chunk)
    uint32_t out_kind;         // OutKind
    uint64_t total_iters;      // MT*NT*KB
};

// LiquidQuant dequantization of one interleaved word (packed.cpp:63-71):
// 2 x LOP3 + SHF to split, 2 x IMAD for q*s+a on four lanes each, 2 x LOP3
// for the XOR 0x80 sign flip. Lane-safe because q*s+a <= 255 for every
// reachable (q, s, a) (quant.hpp:14-16, verify_overflow_free quant.cpp:141).
__device__ __forceinline__ void lqq_dequant_word(uint32_t w, uint32_t s, uint32_t a4,
                                                 uint32_t& lo, uint32_t& hi) {
    lo = ((w & 0x0F0F0F0Fu) * s + a4) ^ 0x80808080u;
    hi = (((w >> 4) & 0x0F0F0F0Fu) * s + a4) ^ 0x80808080u;
}

__device__ __forceinline__ uint64_t cta_range_begin(uint32_t c, uint32_t G, uint64_t total) {
    return total * c / G;
}

// The workspace slot of a split tile = the CTA that owns the tile's first
// k-block. Distinct split tiles have distinct first owners.
__device__ __forceinline__ uint32_t split_slot(uint64_t tile, uint32_t KB, uint32_t G,
                                               uint64_t total) {
    const uint64_t first = tile * KB;
    uint32_t c = static_cast<uint32_t>(first * G / total);
    while (c + 1 < G && cta_range_begin(c + 1, G, total) <= first) ++c;
    while (c > 0 && cta_range_begin(c, G, total) > first) --c;
    return c;
}

__device__ __forceinline__ void store_out(const GemmParams& p, uint32_t m, uint32_t n,
                                          int32_t acc, float cs, float ts) {
    const uint64_t idx = uint64_t(m) * uint64_t(p.ldo) + n;
    if (p.out_kind == kOutAcc) {
        static_cast<int32_t*>(p.out)[idx] = acc;
        return;
    }
    // quant.cpp:125-127: float(double(acc) * double(cs) * double(ts)), left to right.
    const double yd = __dmul_rn(__dmul_rn(double(acc), double(cs)), double(ts));
    const float y = __double2float_rn(yd);
    if (p.out_kind == kOutF32)
        static_cast<float*>(p.out)[idx] = y;
    else if (p.out_kind == kOutF16)
        static_cast<__half*>(p.out)[idx] = __float2half_rn(y);
    else
        static_cast<__nv_bfloat16*>(p.out)[idx] = __float2bfloat16_rn(y);
}

__global__ void __launch_bounds__(kThreads, 1)
    lqg_w4a8_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the SW128 activation tiles.
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t pad = (1024 - (raw_addr & 1023)) & 1023;
    uint8_t* smem = smem_raw + pad;
    const uint32_t smem_base = raw_addr + pad;

    const uint32_t S = p.stages;
    const uint32_t ring_bytes = S * p.stage_bytes;
    // barriers after the ring
    const uint32_t bar_base = smem_base + ring_bytes;
    auto full_bar = [&](uint32_t s) { return bar_base + 8 * s; };
    auto empty_bar = [&](uint32_t s) { return bar_base + 8 * (kMaxStages + s); };
    auto afull_bar = [&](uint32_t a) { return bar_base + 8 * (2 * kMaxStages + a); };
    auto aempty_bar = [&](uint32_t a) { return bar_base + 8 * (2 * kMaxStages + kAStages + a); };
    auto accfull_bar = [&](uint32_t a) { return bar_base + 8 * (2 * kMaxStages + 2 * kAStages + a); };
    auto accempty_bar = [&](uint32_t a) {
        return bar_base + 8 * (2 * kMaxStages + 2 * kAStages + 2 + a);
    };
    uint8_t* misc = smem + ring_bytes + 8 * (2 * kMaxStages + 2 * kAStages + 4);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(misc);
    volatile uint32_t* epi_flag = reinterpret_cast<volatile uint32_t*>(misc + 16);

    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t G = gridDim.x;
    const uint64_t beg = cta_range_begin(blockIdx.x, G, p.total_iters);
    const uint64_t end = cta_range_begin(blockIdx.x + 1, G, p.total_iters);
    const uint32_t n_local = static_cast<uint32_t>(end - beg);
    const uint32_t KB = p.KB;
    const uint32_t acc_stages = p.BN <= 128 ? 2 : 1;
    const uint32_t acc_stride = p.BN <= 128 ? 128 : 256;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(empty_bar(s), 1);
        }
        for (uint32_t a = 0; a < kAStages; ++a) {
            ptx::mbar_init(afull_bar(a), 4);  // one arrive per dequant warp
            ptx::mbar_init(aempty_bar(a), 1);
        }
        for (uint32_t a = 0; a < 2; ++a) {
            ptx::mbar_init(accfull_bar(a), 1);
            ptx::mbar_init(accempty_bar(a), 4);  // one arrive per epilogue warp
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap_x);
    if (warp == 2) ptx::tmem_alloc(ptx::smem_u32(tmem_holder), kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol_w = ptx::policy_evict_first();
            const uint64_t pol_x = ptx::policy_evict_last();
            const uint32_t x_bytes = p.BN * kKBlock;
            for (uint32_t i = 0; i < n_local; ++i) {
                const uint64_t it = beg + i;
                const uint64_t tile = it / KB;
                const uint32_t kb = static_cast<uint32_t>(it % KB);
                const uint32_t mt = static_cast<uint32_t>(tile / p.NT);
                const uint32_t nt = static_cast<uint32_t>(tile % p.NT);
                const uint32_t s = i % S, r = i / S;
                ptx::mbar_wait(empty_bar(s), (r & 1) ^ 1);
                const uint32_t slot = smem_base + s * p.stage_bytes;
                ptx::mbar_arrive_expect_tx(full_bar(s), x_bytes + p.chunk_bytes);
                ptx::tma_2d_g2s(slot, &tmap_x, int32_t(kb * kKBlock), int32_t(mt * p.BN),
                                full_bar(s), pol_x);
                const uint8_t* src = p.wimg + (uint64_t(nt) * KB + kb) * p.chunk_bytes;
                ptx::bulk_g2s(slot + x_bytes, src, p.chunk_bytes, full_bar(s), pol_w);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = ptx::idesc_i8(kTileN, p.BN);
            uint32_t seg = 0;
            for (uint32_t i = 0; i < n_local; ++i) {
                const uint64_t it = beg + i;
                const uint32_t kb = static_cast<uint32_t>(it % KB);
                const bool seg_start = (i == 0) || (kb == 0);
                const bool seg_end = (kb == KB - 1) || (i + 1 == n_local);
                const uint32_t as = seg % acc_stages, ar = seg / acc_stages;
                if (seg_start) {
                    ptx::mbar_wait(accempty_bar(as), (ar & 1) ^ 1);
                    ptx::tc_fence_after();
                }
                const uint32_t s = i % S, a = i % kAStages;
                ptx::mbar_wait(full_bar(s), (i / S) & 1);
                ptx::mbar_wait(afull_bar(a), (i / kAStages) & 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + as * acc_stride;
                const uint32_t a_tmem = tmem_base + kAColBase + a * 32;
                const uint32_t x_addr = smem_base + s * p.stage_bytes;
#pragma unroll
                for (uint32_t k4 = 0; k4 < 4; ++k4) {
                    const uint64_t bdesc = ptx::sw128_kmajor_desc(x_addr + k4 * 32);
                    ptx::mma_i8_ts(d_tmem, a_tmem + k4 * 8, bdesc, idesc,
                                   (seg_start && k4 == 0) ? 0u : 1u);
                }
                ptx::mma_commit(empty_bar(s));
                ptx::mma_commit(aempty_bar(a));
                if (seg_end) {
                    ptx::mma_commit(accfull_bar(as));
                    ++seg;
                }
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ------------------------------------------------------------ dequant WGs
        const uint32_t wg = (warp - 4) / 4;      // 0 or 1: alternate k-blocks
        const uint32_t sp = warp % 4;            // TMEM sub-partition
        const uint32_t row = sp * 32 + lane;     // weight row within the tile = TMEM lane
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t x_bytes = p.BN * kKBlock;
        // sub-block c uses param (c >> p_shift): P=1 -> 2, P=2 -> 1, P=4 -> 0
        const uint32_t p_shift = p.P == 1 ? 2u : (p.P == 2 ? 1u : 0u);
        for (uint32_t i = wg; i < n_local; i += 2) {
            const uint32_t s = i % S, a = i % kAStages;
            ptx::mbar_wait(full_bar(s), (i / S) & 1);
            ptx::mbar_wait(aempty_bar(a), ((i / kAStages) & 1) ^ 1);
            ptx::tc_fence_after();
            const uint8_t* wchunk = smem + s * p.stage_bytes + x_bytes;
            const uint16_t* prm = reinterpret_cast<const uint16_t*>(wchunk + kCodeBytes);
            const uint32_t a_taddr = tmem_base + lane_addr + kAColBase + a * 32;
            uint32_t sa[kSubBlocks];
#pragma unroll
            for (uint32_t c = 0; c < kSubBlocks; ++c) sa[c] = prm[(c >> p_shift) * kTileN + row];
#pragma unroll
            for (uint32_t c = 0; c < kSubBlocks; ++c) {
                const uint32_t sc = sa[c] & 0xFFu;
                const uint32_t a4 = (sa[c] >> 8) * 0x01010101u;
                const uint4 v = *reinterpret_cast<const uint4*>(wchunk + (c * kTileN + row) * 16);
                uint32_t o[8];
                lqq_dequant_word(v.x, sc, a4, o[0], o[1]);
                lqq_dequant_word(v.y, sc, a4, o[2], o[3]);
                lqq_dequant_word(v.z, sc, a4, o[4], o[5]);
                lqq_dequant_word(v.w, sc, a4, o[6], o[7]);
                ptx::tmem_st_x8(a_taddr + c * 8, o);
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(afull_bar(a));
        }
    } else if (warp >= 12) {
        // ------------------------------------------------------------ epilogue
        const uint32_t sp = warp % 4;
        const uint32_t row = sp * 32 + lane;
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t et = threadIdx.x - 12 * 32;  // 0..127
        uint32_t seg = 0;
        uint32_t i = 0;
        while (i < n_local) {
            const uint64_t it = beg + i;
            const uint64_t tile = it / KB;
            const uint32_t kb0 = static_cast<uint32_t>(it % KB);
            const uint32_t n_iters = min(static_cast<uint32_t>(n_local - i), KB - kb0);
            i += n_iters;
            const uint32_t as = seg % acc_stages, ar = seg / acc_stages;
            ++seg;
            const uint32_t mt = static_cast<uint32_t>(tile / p.NT);
            const uint32_t nt = static_cast<uint32_t>(tile % p.NT);
            const uint32_t n = nt * kTileN + row;
            const uint32_t m0 = mt * p.BN;
            const float cs = p.out_kind == kOutAcc ? 0.f : p.cs[n];
            ptx::mbar_wait(accfull_bar(as), ar & 1);
            ptx::tc_fence_after();
            const uint32_t acc_taddr = tmem_base + lane_addr + as * acc_stride;
            const bool whole = (n_iters == KB);
            const uint32_t nchunks = p.BN / 16;
            if (whole) {
                for (uint32_t ch = 0; ch < nchunks; ++ch) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                    ptx::tmem_ld_wait();
                    if (ch + 1 == nchunks) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(accempty_bar(as));
                    }
                    if (n < p.N) {
#pragma unroll
                        for (uint32_t j = 0; j < 16; ++j) {
                            const uint32_t m = m0 + ch * 16 + j;
                            if (m < p.M)
                                store_out(p, m, n, int32_t(v[j]),
                                          cs, p.out_kind == kOutAcc ? 0.f : p.ts[m]);
                        }
                    }
                }
            } else {
                const uint32_t slot = split_slot(tile, KB, G, p.total_iters);
                int32_t* wsl = p.ws + uint64_t(slot) * (256 * kTileN);
                for (uint32_t ch = 0; ch < nchunks; ++ch) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                    ptx::tmem_ld_wait();
                    if (ch + 1 == nchunks) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(accempty_bar(as));
                    }
#pragma unroll
                    for (uint32_t j = 0; j < 16; ++j)
                        atomicAdd(wsl + (ch * 16 + j) * kTileN + row, int32_t(v[j]));
                }
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (et == 0) {
                    const uint32_t old = atomicAdd(p.counters + slot, n_iters);
                    *epi_flag = (old + n_iters == KB) ? 1u : 0u;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                const bool last = *epi_flag != 0;
                if (last) {
                    __threadfence();
                    for (uint32_t mm = 0; mm < p.BN; ++mm) {
                        int32_t* cell = wsl + mm * kTileN + row;
                        const int32_t v = __ldcg(cell);
                        __stcg(cell, 0);
                        const uint32_t m = m0 + mm;
                        if (m < p.M && n < p.N)
                            store_out(p, m, n, v, cs, p.out_kind == kOutAcc ? 0.f : p.ts[m]);
                    }
                    if (et == 0) p.counters[slot] = 0;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc(tmem_base, kTmemCols);
}

}  // namespace lqg
