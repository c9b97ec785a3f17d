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
//   warp 0        TMA producer: per 256-wide k-block, one 1-D bulk copy of
//                 the prepacked weight chunk (codes + group params,
//                 EVICT_FIRST) and two 2-D SW128 tensor copies of the
//                 activation tile (EVICT_LAST) into an S-stage SMEM ring.
//   warp 1        MMA issuer: 8 x tcgen05.mma.kind::i8 (K=32 each) per
//                 k-block, A read from TMEM, B from the swizzled ring slot;
//                 tcgen05.commit frees the ring slot and the TMEM A slot and
//                 signals the epilogue at the end of a tile segment.
//   warp 2        TMEM allocator (512 columns).
//   warps 4-11    two dequant warpgroups (ImFP), each taking half
//                 of every k-block: LDS.128 of packed codes, LiquidQuant
//                 (q*s + a) ^ 0x80 on four byte lanes per IMAD
//                 (packed.cpp:40-61), tcgen05.st of the INT8
//                 result into the TMEM A ring (thread = weight row = lane).
//   warps 12-15   epilogue: tcgen05.ld of the INT32 accumulators, fused
//                 per-channel x per-token scaling and F32/F16/BF16 cast,
//                 coalesced stores (or the INT32 accumulators themselves).
// All hand-offs are mbarrier arrivals (TMA complete_tx, tcgen05.commit,
// thread arrives); there is no __syncthreads in the mainloop.
//
// TMEM (512 columns): [0, acc_stages*acc_stride) INT32 accumulators, then
// the A ring of a_slots x 64 columns (one 256-wide k-block of int8 per slot).
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
constexpr uint32_t kMaxASlots = 4;
constexpr uint32_t kACols = kKBlock / 4;   // TMEM columns per A slot (4 int8 per column)
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kMaxBN = 256;

struct TmemPlan {
    uint32_t acc_stride, acc_stages, a_base, a_slots;
};

__host__ __device__ inline TmemPlan tmem_plan(uint32_t BN) {
    TmemPlan t;
    t.acc_stride = (BN + 31) / 32 * 32;
    t.acc_stages = (2 * t.acc_stride + 2 * kACols <= kTmemCols) ? 2u : 1u;
    t.a_base = (t.acc_stages * t.acc_stride + kACols - 1) / kACols * kACols;
    t.a_slots = (kTmemCols - t.a_base) / kACols;
    if (t.a_slots > kMaxASlots) t.a_slots = kMaxASlots;
    return t;
}

struct GemmParams {
    const uint8_t* wimg;       // prepacked weight image
    const float* cs;           // channel scales (padded to NT*128)
    const float* ts;           // token scales (m)
    void* out;                 // y or acc
    int64_t ldo;               // row pitch of out, in elements
    int32_t* ws;               // split-K workspace: gridDim.x slots of kMaxBN*128 int32
    uint32_t* counters;        // gridDim.x k-block counters
    uint32_t M, N;             // logical problem (tokens, weight rows)
    uint32_t KB, NT, MT;       // k-blocks, weight tiles, token tiles
    uint32_t BN;               // tokens per tile (16..256, multiple of 16)
    uint32_t P;                // group params per k-block (1, 2, 4, 8)
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

// y = float(double(acc) * double(cs) * double(ts)) (quant.cpp:125-127), left
// to right, then the requested cast (RNE). cs_d is double(cs).
__device__ __forceinline__ void store_out(const GemmParams& p, uint32_t m, uint32_t n,
                                          int32_t acc, double cs_d, float ts) {
    const uint64_t idx = uint64_t(m) * uint64_t(p.ldo) + n;
    if (p.out_kind == kOutAcc) {
        static_cast<int32_t*>(p.out)[idx] = acc;
        return;
    }
    const double yd = __dmul_rn(__dmul_rn(double(acc), cs_d), double(ts));
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
    auto aempty_bar = [&](uint32_t a) { return bar_base + 8 * (2 * kMaxStages + kMaxASlots + a); };
    auto accfull_bar = [&](uint32_t a) {
        return bar_base + 8 * (2 * kMaxStages + 2 * kMaxASlots + a);
    };
    auto accempty_bar = [&](uint32_t a) {
        return bar_base + 8 * (2 * kMaxStages + 2 * kMaxASlots + 2 + a);
    };
    uint8_t* misc = smem + ring_bytes + 8 * (2 * kMaxStages + 2 * kMaxASlots + 4);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(misc);
    volatile uint32_t* epi_flag = reinterpret_cast<volatile uint32_t*>(misc + 16);

    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t G = gridDim.x;
    const uint64_t beg = cta_range_begin(blockIdx.x, G, p.total_iters);
    const uint64_t end = cta_range_begin(blockIdx.x + 1, G, p.total_iters);
    const uint32_t n_local = static_cast<uint32_t>(end - beg);
    const uint32_t KB = p.KB;
    const TmemPlan tp = tmem_plan(p.BN);
    const uint32_t x_bytes = p.BN * kKBlock;  // activation tile bytes per stage

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(empty_bar(s), 1);
        }
        for (uint32_t a = 0; a < kMaxASlots; ++a) {
            ptx::mbar_init(afull_bar(a), 8);  // one arrive per dequant warp (both WGs)
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
        const uint64_t pol_w = ptx::policy_evict_first();
        const uint64_t pol_x = ptx::policy_evict_last();
        const uint32_t tx_bytes = x_bytes + p.chunk_bytes;
        const uint32_t atom_bytes = p.BN * kXAtom;
        // incremental (tile, kb) walk: no divisions in the loop
        const uint64_t tile0 = beg / KB;
        uint32_t kb = static_cast<uint32_t>(beg - tile0 * KB);
        uint32_t mt = static_cast<uint32_t>(tile0 / p.NT);
        uint32_t nt = static_cast<uint32_t>(tile0 - uint64_t(mt) * p.NT);
        const uint8_t* src = p.wimg + (uint64_t(nt) * KB + kb) * p.chunk_bytes;
        uint32_t s = 0, ph = 0;
        for (uint32_t i = 0; i < n_local; ++i) {
            ptx::mbar_wait(empty_bar(s), ph ^ 1);
            if (ptx::elect_one()) {
                const uint32_t slot = smem_base + s * p.stage_bytes;
                ptx::mbar_arrive_expect_tx(full_bar(s), tx_bytes);
                const int32_t k0 = int32_t(kb * kKBlock), m0 = int32_t(mt * p.BN);
                ptx::tma_2d_g2s(slot, &tmap_x, k0, m0, full_bar(s), pol_x);
                ptx::tma_2d_g2s(slot + atom_bytes, &tmap_x, k0 + int32_t(kXAtom), m0, full_bar(s),
                                pol_x);
                ptx::bulk_g2s(slot + x_bytes, src, p.chunk_bytes, full_bar(s), pol_w);
            }
            __syncwarp();
            src += p.chunk_bytes;
            if (++kb == KB) {
                kb = 0;
                if (++nt == p.NT) {
                    nt = 0;
                    ++mt;
                    src = p.wimg;
                }
            }
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // The dequant warps wait on full[s] before arriving on afull[a], so
        // afull also orders the TMA-written activation tile before the MMA.
        const uint32_t idesc = ptx::idesc_i8(kTileN, p.BN);
        const uint64_t desc0 = ptx::sw128_kmajor_desc(smem_base);
        const uint32_t stage_desc = p.stage_bytes >> 4;
        const uint32_t atom_desc = (p.BN * kXAtom) >> 4;
        uint32_t kb = static_cast<uint32_t>(beg % KB);
        uint32_t s = 0, a = 0, aph = 0, as = 0, acc_ph = 0;
        for (uint32_t i = 0; i < n_local; ++i) {
            const bool seg_start = (i == 0) || (kb == 0);
            const bool seg_end = (kb == KB - 1) || (i + 1 == n_local);
            if (seg_start) ptx::mbar_wait(accempty_bar(as), acc_ph ^ 1);
            ptx::mbar_wait(afull_bar(a), aph);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint32_t d_tmem = tmem_base + as * tp.acc_stride;
                const uint32_t a_tmem = tmem_base + tp.a_base + a * kACols;
                const uint64_t bdesc = desc0 + uint64_t(s * stage_desc);
#pragma unroll
                for (uint32_t k8 = 0; k8 < kSubBlocks; ++k8)
                    ptx::mma_i8_ts(d_tmem, a_tmem + k8 * 8,
                                   bdesc + (k8 / 4) * atom_desc + (k8 % 4) * 2, idesc,
                                   (seg_start && k8 == 0) ? 0u : 1u);
                ptx::mma_commit(empty_bar(s));
                ptx::mma_commit(aempty_bar(a));
                if (seg_end) ptx::mma_commit(accfull_bar(as));
            }
            __syncwarp();
            if (seg_end && ++as == tp.acc_stages) {
                as = 0;
                acc_ph ^= 1;
            }
            if (++kb == KB) kb = 0;
            if (++s == S) s = 0;
            if (++a == tp.a_slots) {
                a = 0;
                aph ^= 1;
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ------------------------------------------------------------ dequant WGs
        // Both warpgroups work on every k-block: WG w dequantizes sub-blocks
        // [4w, 4w+4). Every waiter therefore observes every phase of every
        // ring barrier (a parity wait can never alias an older phase).
        const uint32_t wg = (warp - 4) / 4;      // 0 or 1: which half of the k-block
        const uint32_t sp = warp % 4;            // TMEM sub-partition
        const uint32_t row = sp * 32 + lane;     // weight row within the tile = TMEM lane
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t p_shift = param_shift(p.P);
        constexpr uint32_t kHalf = kSubBlocks / 2;
        uint32_t s = 0, ph = 0, a = 0, aph = 0;
        const uint8_t* ring_w = smem + x_bytes;
        const uint32_t a_base = tmem_base + lane_addr + tp.a_base + wg * kHalf * 8;
        for (uint32_t i = 0; i < n_local; ++i) {
            ptx::mbar_wait(full_bar(s), ph);
            ptx::mbar_wait(aempty_bar(a), aph ^ 1);
            ptx::tc_fence_after();
            const uint8_t* wchunk = ring_w + s * p.stage_bytes;
            const uint16_t* prm = reinterpret_cast<const uint16_t*>(wchunk + kCodeBytes);
            const uint32_t a_taddr = a_base + a * kACols;
            uint32_t sa[kHalf];
            uint4 v[kHalf];
#pragma unroll
            for (uint32_t cc = 0; cc < kHalf; ++cc) {
                const uint32_t c = wg * kHalf + cc;
                sa[cc] = prm[(c >> p_shift) * kTileN + row];
                v[cc] = *reinterpret_cast<const uint4*>(wchunk + (c * kTileN + row) * 16);
            }
#pragma unroll
            for (uint32_t cc = 0; cc < kHalf; ++cc) {
                const uint32_t sc = sa[cc] & 0xFFu;
                const uint32_t a4 = (sa[cc] >> 8) * 0x01010101u;
                uint32_t o[8];
                lqq_dequant_word(v[cc].x, sc, a4, o[0], o[1]);
                lqq_dequant_word(v[cc].y, sc, a4, o[2], o[3]);
                lqq_dequant_word(v[cc].z, sc, a4, o[4], o[5]);
                lqq_dequant_word(v[cc].w, sc, a4, o[6], o[7]);
                ptx::tmem_st_x8(a_taddr + cc * 8, o);
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(afull_bar(a));
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
            if (++a == tp.a_slots) {
                a = 0;
                aph ^= 1;
            }
        }
    } else if (warp >= 12) {
        // ------------------------------------------------------------ epilogue
        const uint32_t sp = warp % 4;
        const uint32_t row = sp * 32 + lane;
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t et = threadIdx.x - 12 * 32;  // 0..127
        const uint32_t nchunks = p.BN / 16;
        uint32_t as = 0, acc_ph = 0;
        uint32_t i = 0;
        while (i < n_local) {
            const uint64_t it = beg + i;
            const uint64_t tile = it / KB;
            const uint32_t kb0 = static_cast<uint32_t>(it - tile * KB);
            const uint32_t n_iters = min(n_local - i, KB - kb0);
            i += n_iters;
            const uint32_t mt = static_cast<uint32_t>(tile / p.NT);
            const uint32_t nt = static_cast<uint32_t>(tile - uint64_t(mt) * p.NT);
            const uint32_t n = nt * kTileN + row;
            const uint32_t m0 = mt * p.BN;
            const double cs = p.out_kind == kOutAcc ? 0.0 : double(p.cs[n]);
            ptx::mbar_wait(accfull_bar(as), acc_ph);
            ptx::tc_fence_after();
            const uint32_t acc_taddr = tmem_base + lane_addr + as * tp.acc_stride;
            const uint32_t cur_as = as;
            if (++as == tp.acc_stages) {
                as = 0;
                acc_ph ^= 1;
            }
            if (n_iters == KB) {
                // whole tile: scale, cast and store straight from TMEM
                for (uint32_t ch = 0; ch < nchunks; ++ch) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                    ptx::tmem_ld_wait();
                    if (ch + 1 == nchunks) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(accempty_bar(cur_as));
                    }
                    if (n < p.N) {
#pragma unroll
                        for (uint32_t j = 0; j < 16; ++j) {
                            const uint32_t m = m0 + ch * 16 + j;
                            if (m < p.M)
                                store_out(p, m, n, int32_t(v[j]), cs,
                                          p.out_kind == kOutAcc ? 0.f : p.ts[m]);
                        }
                    }
                }
            } else {
                // split tile: exact INT32 reduction through the workspace
                const uint32_t slot = split_slot(tile, KB, G, p.total_iters);
                int32_t* wsl = p.ws + uint64_t(slot) * (kMaxBN * kTileN);
                for (uint32_t ch = 0; ch < nchunks; ++ch) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                    ptx::tmem_ld_wait();
                    if (ch + 1 == nchunks) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(accempty_bar(cur_as));
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
                    for (uint32_t ch = 0; ch < nchunks; ++ch) {
                        int32_t* cell = wsl + ch * 16 * kTileN + row;
                        int32_t v[16];
#pragma unroll
                        for (uint32_t j = 0; j < 16; ++j) v[j] = __ldcg(cell + j * kTileN);
#pragma unroll
                        for (uint32_t j = 0; j < 16; ++j) __stcg(cell + j * kTileN, 0);
                        if (n < p.N) {
#pragma unroll
                            for (uint32_t j = 0; j < 16; ++j) {
                                const uint32_t m = m0 + ch * 16 + j;
                                if (m < p.M)
                                    store_out(p, m, n, v[j], cs,
                                              p.out_kind == kOutAcc ? 0.f : p.ts[m]);
                            }
                        }
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
