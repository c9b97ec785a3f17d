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

// Warp roles: 0 TMA producer, 1 MMA issuer (+ TMEM alloc), then the dequant
// warpgroups, then 4 epilogue warps. One CTA per SM: two dequant WGs (448
// threads). Co-resident decode mode (two CTAs per SM): one dequant WG (320
// threads, so each CTA keeps ~100 registers per thread) -- at BN <= 32 one WG
// dequantizes a k-block several times faster than HBM delivers it.
constexpr uint32_t kThreads = 448;
constexpr uint32_t kDequantWarp0 = 2;
constexpr uint32_t kEpiWarp0 = 10;
template <bool kDecode>
struct Roles {
    static constexpr uint32_t kDQWarps = kDecode ? 4 : 8;
    static constexpr uint32_t kEpi0 = kDequantWarp0 + kDQWarps;
    static constexpr uint32_t kThreadsT = (kEpi0 + 4) * 32;
};
constexpr uint32_t kMaxStages = 16;
constexpr uint32_t kMaxASlots = 8;
constexpr uint32_t kACols = kKBlock / 4;   // TMEM columns per A slot (4 int8 per column)
constexpr uint32_t kMaxBN = 256;
// Token tiles of at most this many 16-token chunks reduce split-K partials
// through registers with sentinel cells; larger ones via flags + TMA gather.
constexpr uint32_t kSentinelMaxChunks = 2;
// Split-K cells per CTA slot: the small-tile region (sentinel protocol, always
// INT32_MIN between launches) first, then the large-tile region (flag
// protocol, contents irrelevant between launches).
constexpr uint32_t kSmallCells = kSentinelMaxChunks * 16 * kTileN;
constexpr uint32_t kSlotCellsK = kSmallCells + kMaxBN * kTileN;

struct TmemPlan {
    uint32_t acc_stride, acc_stages, a_base, a_slots;
};

// cols = allocated TMEM columns: 512 (one CTA per SM) or 256 (decode mode:
// two co-resident CTAs, e.g. consecutive GEMMs overlapped by PDL).
__host__ __device__ inline TmemPlan tmem_plan(uint32_t BN, uint32_t cols) {
    TmemPlan t;
    t.acc_stride = (BN + 31) / 32 * 32;
    t.acc_stages = (2 * t.acc_stride + 2 * kACols <= cols) ? 2u : 1u;
    t.a_base = (t.acc_stages * t.acc_stride + kACols - 1) / kACols * kACols;
    t.a_slots = (cols - t.a_base) / kACols;
    if (t.a_slots > kMaxASlots) t.a_slots = kMaxASlots;
    return t;
}

struct GemmParams {
    const float* ts;           // token scales (all rows)
    void* out;                 // y or acc
    int64_t ldo;               // row pitch of out (and of every fan-out copy), in elements
    void* fan[7];              // extra destinations receiving the same tile (e.g. peer GPUs'
    uint32_t n_fan;            //   Y over NVLink: the fused all-gather of the N-split driver)
    int32_t* parts;            // split-K partials: per CTA kMaxBN*128 int32 cells,
                               // [chunk][quad][row] int4
    uint32_t* flags;           // per CTA: 1 = partial published (release), reset by the finisher
    uint32_t N;                // weight rows
    uint32_t KB, NT, MT;       // k-blocks, weight tiles, token tiles (of the largest group)
    uint32_t BN;               // tokens per tile (16..256, multiple of 16)
    uint32_t P;                // group params per k-block (1, 2, 4, 8)
    uint32_t chunk_bytes;      // bytes per (tile, k-block) weight chunk
    uint32_t stages;           // shared-memory ring depth
    uint32_t stage_bytes;      // bytes per ring slot (X tile first, then W chunk)
    uint32_t out_kind;         // OutKind
    uint32_t tmem_cols;        // 256 (decode mode) or 512
    uint32_t l2_prefetch;      // weight chunks prefetched into L2 ahead of the SMEM ring
    uint32_t w_split;          // bulk copies per weight chunk (1, 2, 4)
    uint32_t dp_rounds;        // whole tiles per CTA before the stream-K tail
    uint32_t raster_gm;        // token tiles per raster group
    uint32_t trace_slot;       // LQG_TRACE builds: launch index % 8
    uint32_t l2_last;          // 1: EVICT_LAST cache hints for reused tiles (default)
    uint32_t pair;             // 1: CTA pairs (cluster of 2, tcgen05 cta_group::2, M = 256):
                               //    NT/tiles count pair tiles, each CTA owns weight tile 2*nt+rank
                               //    and loads half of every activation tile
    uint32_t pdl_trigger;
    uint64_t total_iters;      // tiles*KB
    uint32_t tiles;            // weight-tile x token-tile pairs (summed over groups)
};

// Grouped launch (MoE experts of one layer: same n, k, group size): the
// tiles of every group form one linear space, tile-major within a group.
// Group g owns rows [row0, row0 + M) of X / token scales / Y and tiles
// [tile0, tile0 + MT * NT). A plain GEMM is the one-group case.
struct GroupEntry {
    const uint8_t* wimg;  // prepacked weight image of this group
    const float* cs;      // its channel scales (padded to NT*128)
    uint32_t row0, M, MT, tile0;
};
template <uint32_t kG>
struct GroupTable {
    GroupEntry e[kG];
    uint32_t n;
};
// One tile resolved: its group's weights / scales and its absolute rows.
struct TileRef {
    const uint8_t* wimg;
    const float* cs;
    uint32_t nt, row0, mlim;  // weight tile, first token row, end of the group's rows
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

// CTAs whose range starts strictly inside tile `tile` (its contributors):
// [c_first, c_end). Each contributor's first segment is a piece of the tile.
__device__ __forceinline__ void split_contributors(uint64_t tile, uint32_t KB, uint32_t G,
                                                   uint64_t total, uint32_t& c_first,
                                                   uint32_t& c_end) {
    const uint64_t t0 = tile * KB, t1 = t0 + KB;
    uint32_t c = static_cast<uint32_t>(t0 * G / total);
    while (c > 0 && cta_range_begin(c, G, total) > t0) --c;
    while (c < G && cta_range_begin(c, G, total) <= t0) ++c;
    c_first = c;
    while (c < G && cta_range_begin(c, G, total) < t1) ++c;
    c_end = c;
}

// Hybrid data-parallel + stream-K schedule. With T = MT*NT tiles on G CTAs:
// dp_rounds whole tiles per CTA first (tiles c, c+G, ...; consecutive tile
// indices run concurrently), then a stream-K tail over the remaining
// sk_tiles in [G, 2G) (or all tiles when T < G) so every CTA gets equal work.
// Tiles are rasterized in groups of GM token tiles (n-major inside a group), so
// the ~G tiles in flight share GM activation slices and ~G/GM weight slices
// through L2 instead of spanning the whole M x N grid.
struct Sched {
    uint32_t c, dp_rounds;
    uint32_t sk_tile0, sk_total, sk_beg, sk_end;  // 32-bit: host guarantees total_iters * G < 2^32
    uint32_t sk_tile, sk_kb;                      // first stream-K (tile, k-block) of this CTA
    uint32_t n_local;
};

__device__ __forceinline__ uint32_t range_begin32(uint32_t c, uint32_t G, uint32_t total) {
    return static_cast<uint32_t>((uint64_t(total) * c) / G);
}

// Computed once per CTA (thread 0) and shared through SMEM.
// Scheduling units: CTAs, or CTA pairs (p.pair).
__device__ __forceinline__ uint32_t sched_units(const GemmParams& p) {
    return p.pair ? gridDim.x >> 1 : gridDim.x;
}
__device__ __forceinline__ Sched make_sched(const GemmParams& p) {
    Sched s;
    const uint32_t G = sched_units(p);
    s.c = p.pair ? blockIdx.x >> 1 : blockIdx.x;
    s.dp_rounds = p.dp_rounds;
    s.sk_tile0 = s.dp_rounds * G;
    s.sk_total = (p.tiles - s.sk_tile0) * p.KB;
    s.sk_beg = range_begin32(s.c, G, s.sk_total);
    s.sk_end = range_begin32(s.c + 1, G, s.sk_total);
    s.sk_tile = s.sk_tile0 + s.sk_beg / p.KB;
    s.sk_kb = s.sk_beg % p.KB;
    s.n_local = s.dp_rounds * p.KB + (s.sk_end - s.sk_beg);
    return s;
}

// Position in one CTA's iteration sequence (DP tiles, then its stream-K range).
// Self-contained (KB / dp_rounds come from the kernel parameter bank) so that
// no per-CTA schedule state stays live across the role loops.
// kDP = false (decode mode: dp_rounds == 0) drops the data-parallel phase.
template <bool kDP>
struct Walk {
    uint32_t tile, kb, r, sk_tile, sk_kb;
    __device__ __forceinline__ void init(const Sched& s) {
        r = 0;
        sk_tile = s.sk_tile;
        sk_kb = s.sk_kb;
        if (kDP && s.dp_rounds > 0) {
            tile = s.c;
            kb = 0;
        } else {
            tile = sk_tile;
            kb = sk_kb;
        }
    }
    // Advance one iteration; true if the next iteration is in another tile.
    __device__ __forceinline__ bool next(const GemmParams& p) {
        if (++kb < p.KB) return false;
        kb = 0;
        if (kDP && r < p.dp_rounds) {
            if (++r < p.dp_rounds) {
                tile += sched_units(p);
            } else {
                tile = sk_tile;
                kb = sk_kb;
            }
        } else {
            ++tile;
        }
        return true;
    }
    __device__ __forceinline__ bool in_dp(const GemmParams& p) const { return kDP && r < p.dp_rounds; }
};

// linear tile -> (token tile mt, weight tile nt), from the parameter bank
__device__ __forceinline__ void tile_coords_p(uint32_t t, uint32_t MT, const GemmParams& p,
                                              uint32_t& mt, uint32_t& nt) {
    if (MT == 1) {
        mt = 0;
        nt = t;
        return;
    }
    const uint32_t per_group = p.raster_gm * p.NT;
    const uint32_t g = t / per_group;
    const uint32_t w = t - g * per_group;
    const uint32_t m0 = g * p.raster_gm;
    const uint32_t gm = min(p.raster_gm, MT - m0);
    mt = m0 + w % gm;
    nt = w / gm;
}

template <uint32_t kG>
__device__ __forceinline__ TileRef tile_ref(uint32_t t, const GemmParams& p, const GroupTable<kG>& gt) {
    uint32_t g = 0;
    if (kG > 1)
        while (g + 1 < gt.n && t >= gt.e[g + 1].tile0) ++g;
    const GroupEntry& e = gt.e[g];
    uint32_t mt, nt;
    tile_coords_p(t - e.tile0, e.MT, p, mt, nt);
    TileRef r;
    r.wimg = e.wimg;
    r.cs = e.cs;
    r.nt = p.pair ? 2 * nt + ptx::cluster_ctarank() : nt;
    r.row0 = e.row0 + mt * p.BN;
    r.mlim = e.row0 + e.M;
    return r;
}

// y = float(double(acc) * double(cs) * double(ts)) (quant.cpp:125-127), left
// to right, then the requested cast (RNE). cs_d is double(cs). One call stores
// the 16 tokens [m0, m0+16) of output column n; the output kind is a template
// parameter so every store loop is branch-free (dispatch once per chunk).
// Exact int32 -> double without the conversion unit: 2^52 + 2^31 + acc is
// representable exactly (|acc| < 2^31), so one DADD recovers acc.
__device__ __forceinline__ double i32_to_f64_exact(int32_t a) {
    return __hiloint2double(0x43300000, int(uint32_t(a) ^ 0x80000000u)) - 4503601774854144.0;
}

template <uint32_t kKind, bool kFan>
__device__ __forceinline__ void store_chunk_k(const GemmParams& p, uint32_t m0, uint32_t mlim,
                                              uint32_t n, const int32_t (&acc)[16], double cs_d,
                                              const double* ts) {
    const uint32_t mend = min(16u, mlim > m0 ? mlim - m0 : 0u);
    // one element to the primary output and every fan-out destination
    auto put = [&](uint64_t i, auto v) {
        using T = decltype(v);
        static_cast<T*>(p.out)[i] = v;
        if (kFan)
            for (uint32_t r = 0; r < p.n_fan; ++r) static_cast<T*>(p.fan[r])[i] = v;
    };
    auto one = [&](uint32_t j, uint64_t idx) {
        if (kKind == kOutAcc) {
            put(idx, acc[j]);
        } else {
            const double a = i32_to_f64_exact(acc[j]);
            const float y = __double2float_rn(__dmul_rn(__dmul_rn(a, cs_d), ts[j]));
            if (kKind == kOutF32)
                put(idx, y);
            else if (kKind == kOutF16)
                put(idx, __float2half_rn(y));
            else
                put(idx, __float2bfloat16_rn(y));
        }
    };
    const uint64_t idx0 = uint64_t(m0) * uint64_t(p.ldo) + n;
    if (mend == 16) {
        // full chunk (the common case): branch-free
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j) one(j, idx0 + uint64_t(j) * uint64_t(p.ldo));
    } else {
        // ragged last chunk: same unrolled body under a predicate (static
        // register indices, no local-memory copy of acc)
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j)
            if (j < mend) one(j, idx0 + uint64_t(j) * uint64_t(p.ldo));
    }
}

template <bool kFan>
__device__ __forceinline__ void store_chunk(const GemmParams& p, uint32_t m0, uint32_t mlim, uint32_t n,
                                            const int32_t (&acc)[16], double cs_d, const double* ts) {
    switch (p.out_kind) {
        case kOutAcc: store_chunk_k<kOutAcc, kFan>(p, m0, mlim, n, acc, cs_d, ts); break;
        case kOutF32: store_chunk_k<kOutF32, kFan>(p, m0, mlim, n, acc, cs_d, ts); break;
        case kOutF16: store_chunk_k<kOutF16, kFan>(p, m0, mlim, n, acc, cs_d, ts); break;
        default: store_chunk_k<kOutBF16, kFan>(p, m0, mlim, n, acc, cs_d, ts); break;
    }
}

#ifdef LQG_TRACE
__device__ unsigned long long g_lqg_trace[8 * 160 * 16];
__device__ __forceinline__ void trace(uint32_t slot, uint32_t e) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_lqg_trace[(slot * 160 + blockIdx.x) * 16 + e] = t;
}
#define LQG_T(e) trace(p.trace_slot, e)
#define LQG_TV(e, v) (g_lqg_trace[(p.trace_slot * 160 + blockIdx.x) * 16 + (e)] = (v))
#else
#define LQG_T(e) ((void)0)
#define LQG_TV(e, v) ((void)0)
#endif

// kDecode: two CTAs per SM (<= 110 KB SMEM, 256 TMEM columns, <= 72 registers)
// so consecutive GEMMs overlap under PDL; otherwise one CTA per SM.
// kG > 1: grouped launch over up to kG weight groups (MoE experts).
// kFan: the epilogue also stores every tile into p.fan[0..n_fan) (fused
// all-gather of the N-split driver); a separate instantiation so the plain
// kernel's epilogue is untouched.
// kPair: CTA pairs (cluster of two, tcgen05 cta_group::2, M = 256): each
// CTA dequantizes its own 128 weight rows into its TMEM and loads half of the
// activation tile (N/2 tokens); the leader issues one M=256 MMA that reads the
// B halves from both CTAs' shared memory, which halves the activation
// shared-memory traffic per SM (the bound at large M).
template <bool kDecode, uint32_t kG, bool kFan, bool kPair = false>
__global__ void __launch_bounds__(Roles<kDecode>::kThreadsT, kDecode ? 2 : 1)
    lqg_w4a8_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const GemmParams p,
                         const __grid_constant__ GroupTable<kG> gt) {
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
    auto wfull_bar = [&](uint32_t s) { return bar_base + 8 * s; };
    auto xfull_bar = [&](uint32_t s) { return bar_base + 8 * (kMaxStages + s); };
    auto empty_bar = [&](uint32_t s) { return bar_base + 8 * (2 * kMaxStages + s); };
    constexpr uint32_t kB = 3 * kMaxStages;
    auto afull_bar = [&](uint32_t a) { return bar_base + 8 * (kB + a); };
    auto aempty_bar = [&](uint32_t a) { return bar_base + 8 * (kB + kMaxASlots + a); };
    auto accfull_bar = [&](uint32_t a) { return bar_base + 8 * (kB + 2 * kMaxASlots + a); };
    auto accempty_bar = [&](uint32_t a) { return bar_base + 8 * (kB + 2 * kMaxASlots + 2 + a); };
    const uint32_t fin_bar = bar_base + 8 * (kB + 2 * kMaxASlots + 4);  // split-K gather (finisher)
    uint8_t* misc = smem + ring_bytes + 8 * (kB + 2 * kMaxASlots + 5);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(misc);
    double* ts_s = reinterpret_cast<double*>(misc + 128);  // kMaxBN token scales, as double

    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t G = sched_units(p);
    Sched* sched_s = reinterpret_cast<Sched*>(misc + 32);
    const uint32_t KB = p.KB;
    const TmemPlan tp = tmem_plan(p.BN, p.tmem_cols);
    const uint32_t rank = kPair ? ptx::cluster_ctarank() : 0u;  // 0 = pair leader
    // activation bytes this CTA loads per stage (half of the tile in a pair)
    const uint32_t x_bytes = (kPair ? p.BN / 2 : p.BN) * kKBlock;
    // barriers the pair leader waits on, as seen from this CTA
    auto leader = [&](uint32_t bar) { return kPair ? ptx::mapa(bar, 0) : bar; };

    if (threadIdx.x == 0) LQG_T(0);
    if (threadIdx.x == 0) {
        *sched_s = make_sched(p);
        for (uint32_t s = 0; s < S; ++s) {
            ptx::mbar_init(wfull_bar(s), 1);
            ptx::mbar_init(xfull_bar(s), 1);
            ptx::mbar_init(empty_bar(s), 1);
        }
        for (uint32_t a = 0; a < kMaxASlots; ++a) {
            ptx::mbar_init(afull_bar(a), (kPair ? 2 : 1) * Roles<kDecode>::kDQWarps);  // one arrive per dequant warp
            ptx::mbar_init(aempty_bar(a), 1);
        }
        for (uint32_t a = 0; a < 2; ++a) {
            ptx::mbar_init(accfull_bar(a), 1);
            ptx::mbar_init(accempty_bar(a), kPair ? 8 : 4);  // one arrive per epilogue warp
        }
        ptx::mbar_init(fin_bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap_x);
    if (warp == 1) {
        if (kPair)
            ptx::tmem_alloc_pair(ptx::smem_u32(tmem_holder), p.tmem_cols);
        else
            ptx::tmem_alloc(ptx::smem_u32(tmem_holder), p.tmem_cols);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (kPair) ptx::cluster_sync();  // the peer's barriers are initialised before any remote arrive
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const Sched sch = *sched_s;
    const uint32_t n_local = sch.n_local;
    // PDL: let the next kernel in the stream start its prologue and weight
    // prefetch now; everything that reads or writes dependent memory below
    // (activations, token scales, outputs, workspace) sits behind
    // griddepcontrol.wait.
    if (threadIdx.x == 0 && p.pdl_trigger == 0) ptx::launch_dependents();
    if (threadIdx.x == 0) LQG_T(1);

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        // Weights (static) are streamed immediately: the first min(S, n)
        // chunks are in flight before griddepcontrol.wait, so the weight
        // stream of this GEMM overlaps the tail of the previous kernel.
        // Activation tiles follow the dependency wait.
        // Reused tiles (activations; weights re-read by several token tiles)
        // EVICT_LAST, a single-pass weight stream EVICT_FIRST. (Normal
        // priority via LQG_L2_EVICT_LAST=0 measured ~2 % slower at M = 4096.)
        const uint64_t pol_w = p.MT == 1 ? ptx::policy_evict_first()
                                         : (p.l2_last ? ptx::policy_evict_last() : ptx::policy_evict_normal());
        const uint64_t pol_x = p.l2_last ? ptx::policy_evict_last() : ptx::policy_evict_normal();
        const uint32_t atom_bytes = (kPair ? p.BN / 2 : p.BN) * kXAtom;
        // weight walker
        Walk<!kDecode> ww;
        ww.init(sch);
        auto chunk_src = [&](uint32_t tile, uint32_t kb) {
            const TileRef r = tile_ref(tile, p, gt);
            return r.wimg + (uint64_t(r.nt) * KB + kb) * p.chunk_bytes;
        };
        const uint8_t* src = chunk_src(ww.tile, ww.kb);
        auto w_next = [&]() {
            if (ww.next(p)) {
                src = chunk_src(ww.tile, ww.kb);
            } else {
                src += p.chunk_bytes;
            }
        };
        // weight chunk -> SMEM as w_split concurrent bulk copies (16-byte granular)
        const uint32_t part = (p.chunk_bytes / p.w_split + 15) / 16 * 16;
        auto w_copy = [&](uint32_t dst, const uint8_t* gsrc, uint32_t bar) {
            for (uint32_t off = 0; off < p.chunk_bytes; off += part)
                ptx::bulk_g2s(dst + off, gsrc + off, min(part, p.chunk_bytes - off), bar, pol_w);
        };
        // activation walker
        Walk<!kDecode> xw;
        xw.init(sch);
        uint32_t xrow0 = tile_ref(xw.tile, p, gt).row0;
        auto x_issue = [&](uint32_t st) {
            const uint32_t slot = smem_base + st * p.stage_bytes;
#ifdef LQG_EXP_NOXTMA
            ptx::mbar_arrive(xfull_bar(st));  // timing experiment: no activation traffic
            return;
#endif
            const int32_t k0 = int32_t(xw.kb * kKBlock);
            if (kPair) {
                // both halves count on the leader's barrier; the leader expects the whole tile
                if (rank == 0) ptx::mbar_arrive_expect_tx(xfull_bar(st), 2 * x_bytes);
                const int32_t m0 = int32_t(xrow0 + rank * (p.BN / 2));
                const uint32_t fb = ptx::mapa(xfull_bar(st), 0);
                ptx::tma_2d_g2s_pair(slot, &tmap_x, k0, m0, fb, pol_x);
                ptx::tma_2d_g2s_pair(slot + atom_bytes, &tmap_x, k0 + int32_t(kXAtom), m0, fb, pol_x);
                return;
            }
            ptx::mbar_arrive_expect_tx(xfull_bar(st), x_bytes);
            const int32_t m0 = int32_t(xrow0);
            ptx::tma_2d_g2s(slot, &tmap_x, k0, m0, xfull_bar(st), pol_x);
            ptx::tma_2d_g2s(slot + atom_bytes, &tmap_x, k0 + int32_t(kXAtom), m0, xfull_bar(st),
                            pol_x);
        };
        auto x_next = [&]() {
            if (xw.next(p)) xrow0 = tile_ref(xw.tile, p, gt).row0;
        };
        const uint32_t pre = n_local < S ? n_local : S;
        for (uint32_t i = 0; i < pre; ++i) {
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(wfull_bar(i), p.chunk_bytes);
                w_copy(smem_base + i * p.stage_bytes + x_bytes, src, wfull_bar(i));
            }
            __syncwarp();
            w_next();
        }
        // L2 prefetch stream, D = p.l2_prefetch chunks ahead of the SMEM ring:
        // DRAM latency is covered by L2-resident chunks, so the SMEM ring only
        // has to cover L2 latency (decode mode keeps it small for co-residency).
        // The first D chunks are requested before the PDL wait, so HBM keeps
        // streaming this GEMM's weights while the previous kernel drains.
        Walk<!kDecode> fw = ww;
        const uint8_t* fsrc = src;
        uint32_t pf_issued = pre;  // chunks [pre, pf_issued) requested so far
        auto pf_next = [&]() {
            if (fw.next(p)) {
                fsrc = chunk_src(fw.tile, fw.kb);
            } else {
                fsrc += p.chunk_bytes;
            }
        };
        for (; pf_issued < min(n_local, pre + p.l2_prefetch); ++pf_issued) {
            if (ptx::elect_one()) ptx::prefetch_l2(fsrc, p.chunk_bytes);
            __syncwarp();
            pf_next();
        }
        ptx::griddep_wait();
        if (lane == 0) LQG_T(2);
        for (uint32_t i = 0; i < pre; ++i) {
            if (ptx::elect_one()) x_issue(i);
            __syncwarp();
            x_next();
        }
        uint32_t s = pre == S ? 0 : pre, ph = pre == S ? 1 : 0;
        for (uint32_t i = pre; i < n_local; ++i) {
            ptx::mbar_wait(empty_bar(s), ph ^ 1);
            if (ptx::elect_one()) {
#ifdef LQG_EXP_NOWTMA
                ptx::mbar_arrive(wfull_bar(s));
#else
                ptx::mbar_arrive_expect_tx(wfull_bar(s), p.chunk_bytes);
                w_copy(smem_base + s * p.stage_bytes + x_bytes, src, wfull_bar(s));
#endif
                x_issue(s);
                if (pf_issued < n_local) ptx::prefetch_l2(fsrc, p.chunk_bytes);
            }
            __syncwarp();
            if (pf_issued < n_local) {
                ++pf_issued;
                pf_next();
            }
            w_next();
            x_next();
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
        }
        if (lane == 0 && p.pdl_trigger == 1) ptx::launch_dependents();
    } else if (warp == 1 && (!kPair || rank == 0)) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = ptx::idesc_i8(kPair ? 2 * kTileN : kTileN, p.BN);
        const uint64_t desc0 = ptx::sw128_kmajor_desc(smem_base);
        const uint32_t stage_desc = p.stage_bytes >> 4;
        const uint32_t atom_desc = ((kPair ? p.BN / 2 : p.BN) * kXAtom) >> 4;
        Walk<!kDecode> mw;
        mw.init(sch);
        bool seg_start = true;
        uint32_t s = 0, ph = 0, a = 0, aph = 0, as = 0, acc_ph = 0;
#ifdef LQG_TRACE
        long long w_acc = 0, w_a = 0, w_x = 0;
        const long long t_mma0 = clock64();
#endif
        for (uint32_t i = 0; i < n_local; ++i) {
            const bool seg_end = (mw.kb == KB - 1) || (i + 1 == n_local);
#ifdef LQG_TRACE
            const long long tw0 = clock64();
            if (seg_start) ptx::mbar_wait(accempty_bar(as), acc_ph ^ 1);
            const long long tw1 = clock64();
            ptx::mbar_wait(afull_bar(a), aph);
            const long long tw2 = clock64();
            ptx::mbar_wait(xfull_bar(s), ph);
            const long long tw3 = clock64();
            w_acc += tw1 - tw0;
            w_a += tw2 - tw1;
            w_x += tw3 - tw2;
#else
            if (seg_start) ptx::mbar_wait(accempty_bar(as), acc_ph ^ 1);
            ptx::mbar_wait(afull_bar(a), aph);
            ptx::mbar_wait(xfull_bar(s), ph);
#endif
#ifndef LQG_TRACE_DQ
            if (i == 0 && lane == 0) LQG_T(4);
            if (i + 1 == n_local && lane == 0) LQG_T(5);
#endif
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint32_t d_tmem = tmem_base + as * tp.acc_stride;
                const uint32_t a_tmem = tmem_base + tp.a_base + a * kACols;
                const uint64_t bdesc = desc0 + uint64_t(s * stage_desc);
#pragma unroll
                for (uint32_t k8 = 0; k8 < kSubBlocks; ++k8)
                    if (kPair)
                        ptx::mma_i8_ts_pair(d_tmem, a_tmem + k8 * 8,
                                            bdesc + (k8 / 4) * atom_desc + (k8 % 4) * 2, idesc,
                                            (seg_start && k8 == 0) ? 0u : 1u);
                    else
                        ptx::mma_i8_ts(d_tmem, a_tmem + k8 * 8,
                                       bdesc + (k8 / 4) * atom_desc + (k8 % 4) * 2, idesc,
                                       (seg_start && k8 == 0) ? 0u : 1u);
                if (kPair) {
                    ptx::mma_commit_pair(empty_bar(s));
                    ptx::mma_commit_pair(aempty_bar(a));
                    if (seg_end) ptx::mma_commit_pair(accfull_bar(as));
                } else {
                    ptx::mma_commit(empty_bar(s));
                    ptx::mma_commit(aempty_bar(a));
                    if (seg_end) ptx::mma_commit(accfull_bar(as));
                }
            }
            __syncwarp();
            if (seg_end && ++as == tp.acc_stages) {
                as = 0;
                acc_ph ^= 1;
            }
            seg_start = mw.next(p);
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
            if (++a == tp.a_slots) {
                a = 0;
                aph ^= 1;
            }
        }
        if (lane == 0 && p.pdl_trigger == 2) ptx::launch_dependents();
#ifdef LQG_TRACE
        if (lane == 0) {  // MMA-warp wait cycles: accumulator, A operand, activation tile, total
            LQG_TV(12, (unsigned long long)w_acc);
            LQG_TV(13, (unsigned long long)w_a);
            LQG_TV(14, (unsigned long long)w_x);
            LQG_TV(15, (unsigned long long)(clock64() - t_mma0));
        }
#endif
    } else if (warp >= kDequantWarp0 && warp < Roles<kDecode>::kEpi0) {
        // ------------------------------------------------------------ dequant WGs
        // Both warpgroups work on every k-block: WG w dequantizes sub-blocks
        // [4w, 4w+4). Every waiter therefore observes every phase of every
        // ring barrier (a parity wait can never alias an older phase).
        const uint32_t wg = (warp - kDequantWarp0) / 4;  // which part of the k-block
        const uint32_t sp = warp % 4;            // TMEM sub-partition
        const uint32_t row = sp * 32 + lane;     // weight row within the tile = TMEM lane
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t p_shift = param_shift(p.P);
        constexpr uint32_t kHalf = kSubBlocks / (Roles<kDecode>::kDQWarps / 4);  // sub-blocks per WG
        uint32_t s = 0, ph = 0, a = 0, aph = 0;
#ifdef LQG_TRACE
        long long dq_w = 0, dq_a = 0, dq_st = 0, dq_ar = 0;
        const long long t_dq0 = clock64();
#endif
        const uint8_t* ring_w = smem + x_bytes;
        const uint32_t a_base = tmem_base + lane_addr + tp.a_base + wg * kHalf * 8;
        for (uint32_t i = 0; i < n_local; ++i) {
#ifdef LQG_TRACE
            const long long td0 = clock64();
            ptx::mbar_wait(wfull_bar(s), ph);
            const long long td1 = clock64();
            ptx::mbar_wait(aempty_bar(a), aph ^ 1);
            const long long td2 = clock64();
            dq_w += td1 - td0;
            dq_a += td2 - td1;
#else
            ptx::mbar_wait(wfull_bar(s), ph);
            ptx::mbar_wait(aempty_bar(a), aph ^ 1);
#endif
            ptx::tc_fence_after();
            const uint8_t* wchunk = ring_w + s * p.stage_bytes;
            const uint16_t* prm = reinterpret_cast<const uint16_t*>(wchunk + kCodeBytes);
            const uint32_t a_taddr = a_base + a * kACols;
            uint32_t sa[kHalf];
            uint4 v[kHalf];
#pragma unroll
            for (uint32_t cc = 0; cc < kHalf; ++cc) {
                const uint32_t c = wg * kHalf + cc;
#ifdef LQG_EXP_NOLDS
                sa[cc] = 0x8001u + c;
                v[cc] = make_uint4(row, c, i, s);
                (void)prm;
                (void)wchunk;
#else
                sa[cc] = prm[(c >> p_shift) * kTileN + row];
                v[cc] = *reinterpret_cast<const uint4*>(wchunk + (c * kTileN + row) * 16);
#endif
            }
#pragma unroll
            for (uint32_t cc = 0; cc < kHalf; ++cc) {
                const uint32_t sc = sa[cc] & 0xFFu;
                const uint32_t a4 = (sa[cc] >> 8) * 0x01010101u;
                uint32_t o[8];
#ifdef LQG_EXP_NODEQUANT
                o[0] = v[cc].x; o[1] = v[cc].y; o[2] = v[cc].z; o[3] = v[cc].w;
                o[4] = sc; o[5] = a4; o[6] = v[cc].x; o[7] = v[cc].y;
#else
                lqq_dequant_word(v[cc].x, sc, a4, o[0], o[1]);
                lqq_dequant_word(v[cc].y, sc, a4, o[2], o[3]);
                lqq_dequant_word(v[cc].z, sc, a4, o[4], o[5]);
                lqq_dequant_word(v[cc].w, sc, a4, o[6], o[7]);
#endif
                ptx::tmem_st_x8(a_taddr + cc * 8, o);
            }
#ifdef LQG_TRACE
            const long long td3 = clock64();
#endif
            ptx::tmem_st_wait();
#ifdef LQG_TRACE
            const long long td4 = clock64();
#endif
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (kPair && rank != 0)
                    ptx::mbar_arrive_cluster_relaxed(leader(afull_bar(a)));
                else
                    ptx::mbar_arrive(afull_bar(a));
            }
#ifdef LQG_TRACE
            __syncwarp();
            dq_st += td4 - td3;
            dq_ar += clock64() - td4;
#endif
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
            if (++a == tp.a_slots) {
                a = 0;
                aph ^= 1;
            }
        }
#ifdef LQG_TRACE_DQ  // (with LQG_TRACE) replaces the timeline slots 2-5 and 11
        if (warp == kDequantWarp0 && lane == 0) {  // dequant waits: weights, A slot, total
            LQG_TV(2, (unsigned long long)dq_w);
            LQG_TV(3, (unsigned long long)dq_a);
            LQG_TV(4, (unsigned long long)dq_st);
            LQG_TV(5, (unsigned long long)dq_ar);
            LQG_TV(11, (unsigned long long)(clock64() - t_dq0));
        }
#endif
    } else if (warp >= Roles<kDecode>::kEpi0) {
        // ------------------------------------------------------------ epilogue
        const uint32_t sp = warp % 4;
        const uint32_t row = sp * 32 + lane;
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t et = threadIdx.x - Roles<kDecode>::kEpi0 * 32;  // 0..127
        const uint32_t nchunks = p.BN / 16;
        const bool scaled = p.out_kind != kOutAcc;
        ptx::griddep_wait();
        uint32_t as = 0, acc_ph = 0, fin_ph = 0;
        uint32_t i = 0;
        Walk<!kDecode> ew;
        ew.init(sch);
        while (i < n_local) {
            const uint32_t tile = ew.tile;
            const uint32_t kb0 = ew.kb;
            const uint32_t n_iters = ew.in_dp(p) ? KB : min(n_local - i, KB - kb0);
            i += n_iters;
            ew.kb = KB - 1;  // jump to the start of the next segment
            ew.next(p);
            const TileRef tr = tile_ref(tile, p, gt);
            const uint32_t n = tr.nt * kTileN + row;
            const uint32_t m0 = tr.row0, mlim = tr.mlim;
            // Scales are fetched while the MMAs of this segment are in flight:
            // the token scales of the tile go to shared memory (read back as
            // broadcasts), the channel scale of this thread's row to a register.
            const double cs = scaled ? double(tr.cs[n]) : 0.0;
            if (scaled)
                for (uint32_t j = et; j < p.BN; j += 128)
                    ts_s[j] = m0 + j < mlim ? double(p.ts[m0 + j]) : 0.0;
            // Head piece of a split tile: find its contributors now, while this
            // segment's MMAs run; for small token tiles also request the first
            // batch's chunk-0 cells (they are usually published by now).
            const bool finisher = n_iters < KB && kb0 == 0;
            const bool small = nchunks <= kSentinelMaxChunks;
            uint32_t c_first = 0, c_end = 0;
            // Split-K cells of up to four contributors for one 16-token chunk:
            // [contributor][quad]. Loaded one chunk ahead (software pipeline).
            int4 cb[4][4];
            auto cell_of = [&](uint32_t c, uint32_t ch) {
                const uint32_t cs_slot = kPair ? 2 * c + rank : c;  // the matching CTA of a contributor pair
                return reinterpret_cast<int4*>(p.parts + uint64_t(cs_slot) * kSlotCellsK + (small ? 0u : kSmallCells)) +
                       ch * 4 * kTileN + row;
            };
            auto load_batch = [&](uint32_t c, uint32_t ch) {
                const uint32_t nb = min(4u, c_end - c);
#pragma unroll
                for (uint32_t b = 0; b < 4; ++b)
                    if (b < nb)
#pragma unroll
                        for (uint32_t q = 0; q < 4; ++q) cb[b][q] = __ldcg(cell_of(c + b, ch) + q * kTileN);
            };
            if (finisher) {
                split_contributors(uint64_t(tile - sch.sk_tile0), KB, G, sch.sk_total, c_first, c_end);
                if (small) load_batch(c_first, 0);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            ptx::mbar_wait_parked(accfull_bar(as), acc_ph);  // idle for a tile mainloop
            if (i >= n_local && et == 0) LQG_T(6);
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
                        if (lane == 0) {
                            if (kPair && rank != 0)
                                ptx::mbar_arrive_cluster_relaxed(leader(accempty_bar(cur_as)));
                            else
                                ptx::mbar_arrive(accempty_bar(cur_as));
                        }
                    }
                    if (n < p.N) {
                        int32_t a[16];
#pragma unroll
                        for (uint32_t j = 0; j < 16; ++j) a[j] = int32_t(v[j]);
                        store_chunk<kFan>(p, m0 + ch * 16, mlim, n, a, cs, ts_s + ch * 16);
                    }
                }
            } else if (kb0 > 0) {
                // Contributor piece of a split tile (always this CTA's first
                // segment): publish the INT32 partial into this CTA's cells.
                // Small tiles: no fence and no flag -- |partial| <= 133120 *
                // 127^2 < 2^31, so INT32_MIN never occurs as a value and marks
                // "not published". Large tiles: a release flag per CTA.
                int32_t* slot = p.parts + uint64_t(blockIdx.x) * kSlotCellsK + (small ? 0u : kSmallCells);
                for (uint32_t ch = 0; ch < nchunks; ++ch) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                    ptx::tmem_ld_wait();
                    if (ch + 1 == nchunks) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if (kPair && rank != 0)
                                ptx::mbar_arrive_cluster_relaxed(leader(accempty_bar(cur_as)));
                            else
                                ptx::mbar_arrive(accempty_bar(cur_as));
                        }
                    }
                    // [chunk][quad q][row] int4 cells: a warp's stores are 512
                    // contiguous bytes, and the finisher's bulk copy is one block
                    int4* cell = reinterpret_cast<int4*>(slot) + ch * 4 * kTileN + row;
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q)
                        __stcg(cell + q * kTileN, make_int4(int32_t(v[4 * q]), int32_t(v[4 * q + 1]),
                                                            int32_t(v[4 * q + 2]), int32_t(v[4 * q + 3])));
                }
                if (nchunks > kSentinelMaxChunks) {
                    // large tiles: every epilogue thread's stores, then one release flag
                    __threadfence();
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (et == 0) ptx::st_release_u32(p.flags + blockIdx.x, 1u);
                }
                if (et == 0) LQG_T(9);
            } else {
                // Head piece of a split tile: this CTA finishes the tile (in
                // stream-K order it is the CTA's last segment). Integer addition
                // is associative: bit-exact in any arrival order. Between
                // launches every small-region cell holds the sentinel and every
                // flag is 0.
                if (small) {
                    // Small token tiles (<= 2 chunks): the contributors' cells come
                    // straight into registers, four contributors per L2 round
                    // trip, the first batch requested before the accumulator wait
                    // and the next chunk's one chunk ahead; cells still holding
                    // the sentinel are re-read until published, then reset.
                    for (uint32_t ch = 0; ch < nchunks; ++ch) {
                        uint32_t v[16];
                        ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                        ptx::tmem_ld_wait();
                        int32_t sum[16];
#pragma unroll
                        for (uint32_t j = 0; j < 16; ++j) sum[j] = int32_t(v[j]);
                        for (uint32_t c = c_first; c < c_end; c += 4) {
                            const uint32_t nb = min(4u, c_end - c);
                            if (c != c_first) load_batch(c, ch);
                            auto pend = [](const int4& x) {
                                return x.x == INT32_MIN || x.y == INT32_MIN || x.z == INT32_MIN ||
                                       x.w == INT32_MIN;
                            };
                            for (;;) {
                                uint32_t mask = 0;
#pragma unroll
                                for (uint32_t b = 0; b < 4; ++b)
#pragma unroll
                                    for (uint32_t q = 0; q < 4; ++q)
                                        mask |= (b < nb && pend(cb[b][q])) ? (1u << (4 * b + q)) : 0u;
                                if (!mask) break;
                                __nanosleep(32);
#pragma unroll
                                for (uint32_t b = 0; b < 4; ++b)
#pragma unroll
                                    for (uint32_t q = 0; q < 4; ++q)
                                        if (mask & (1u << (4 * b + q)))
                                            cb[b][q] = ptx::ld_relaxed_v4(cell_of(c + b, ch) + q * kTileN);
                            }
#pragma unroll
                            for (uint32_t b = 0; b < 4; ++b) {
                                if (b < nb) {
#pragma unroll
                                    for (uint32_t q = 0; q < 4; ++q) {
                                        sum[4 * q] += cb[b][q].x;
                                        sum[4 * q + 1] += cb[b][q].y;
                                        sum[4 * q + 2] += cb[b][q].z;
                                        sum[4 * q + 3] += cb[b][q].w;
                                        __stcg(cell_of(c + b, ch) + q * kTileN,
                                               make_int4(INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN));
                                    }
                                }
                            }
                            if (c + 4 >= c_end && ch + 1 < nchunks) load_batch(c_first, ch + 1);
                        }
                        if (n < p.N) store_chunk<kFan>(p, m0 + ch * 16, mlim, n, sum, cs, ts_s + ch * 16);
                    }
                } else {
                    // Large token tiles: this is the CTA's last segment, so the
                    // SMEM ring is idle. Wait (acquire) until every contributor
                    // has raised its flag, then gather the partials (one
                    // contiguous BN*512-byte block each) by TMA bulk copies, as
                    // many per batch as the ring holds, and sum them from SMEM:
                    // two L2 round trips per batch instead of one per 16-token
                    // chunk. Flags are reset for the next launch (which touches
                    // them only after griddepcontrol.wait).
                    const uint32_t part_bytes = p.BN * kTileN * 4;
                    const uint32_t nb_max = max(1u, ring_bytes / part_bytes);
                    const int4* sm4 = reinterpret_cast<const int4*>(smem);
                    for (uint32_t c = c_first + et; c < c_end; c += 128) {
                        const uint32_t fc = kPair ? 2 * c + rank : c;
                        while (ptx::ld_acquire_u32(p.flags + fc) == 0) __nanosleep(32);
                        p.flags[fc] = 0;
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    (void)0;
                    for (uint32_t c0 = c_first; c0 < c_end; c0 += nb_max) {
                        const uint32_t nb = min(nb_max, c_end - c0);
                        const bool last_batch = c0 + nb >= c_end;
                        if (et == 0) {
                            ptx::fence_proxy_async();  // acquired data + prior generic SMEM reads vs TMA
                            ptx::mbar_arrive_expect_tx(fin_bar, nb * part_bytes);
                            for (uint32_t b = 0; b < nb; ++b)
                                ptx::bulk_g2s(smem_base + b * part_bytes,
                                              p.parts + uint64_t(kPair ? 2 * (c0 + b) + rank : c0 + b) * kSlotCellsK + kSmallCells, part_bytes,
                                              fin_bar, ptx::policy_evict_first());
                        }
                        ptx::mbar_wait(fin_bar, fin_ph);
                        fin_ph ^= 1;
                        for (uint32_t ch = 0; ch < nchunks; ++ch) {
                            uint32_t v[16];
                            ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                            ptx::tmem_ld_wait();
                            int32_t sum[16];
#pragma unroll
                            for (uint32_t j = 0; j < 16; ++j) sum[j] = int32_t(v[j]);
                            for (uint32_t b = 0; b < nb; ++b) {
                                const int4* scell = sm4 + b * (part_bytes / 16) + ch * 4 * kTileN + row;
#pragma unroll
                                for (uint32_t q = 0; q < 4; ++q) {
                                    const int4 x = scell[q * kTileN];
                                    sum[4 * q] += x.x;
                                    sum[4 * q + 1] += x.y;
                                    sum[4 * q + 2] += x.z;
                                    sum[4 * q + 3] += x.w;
                                }
                            }
                            if (!last_batch) {
                                // running sum back into the accumulator for the next batch
                                ptx::tmem_st_x16(acc_taddr + ch * 16, sum);
                            } else {
                                if (ch == 0 && et == 0) LQG_T(10);
                                if (n < p.N) store_chunk<kFan>(p, m0 + ch * 16, mlim, n, sum, cs, ts_s + ch * 16);
                            }
                        }
                        if (!last_batch) ptx::tmem_st_wait();
                        asm volatile("bar.sync 1, 128;" ::: "memory");  // ring reads done before the next batch
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                            if (kPair && rank != 0)
                                ptx::mbar_arrive_cluster_relaxed(leader(accempty_bar(cur_as)));
                            else
                                ptx::mbar_arrive(accempty_bar(cur_as));
                        }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");  // ts_s reuse
        }
    }

    if (warp == Roles<kDecode>::kEpi0 && lane == 0) LQG_T(7);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) LQG_T(8);
    if (kPair) ptx::cluster_sync();  // the leader's MMAs into this CTA's TMEM are complete
    if (warp == 1) {
        if (kPair)
            ptx::tmem_dealloc_pair(tmem_base, p.tmem_cols);
        else
            ptx::tmem_dealloc(tmem_base, p.tmem_cols);
    }
}

}  // namespace lqg
