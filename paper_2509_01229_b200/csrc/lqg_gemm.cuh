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
// Warp roles in one 480-thread CTA (one CTA per SM, persistent, stream-K):
//   warp 0        W producer: per 256-wide k-block one 1-D bulk copy of the
//                 prepacked weight chunk (codes + group params) into the
//                 W ring. The first ring of chunks is requested before
//                 griddepcontrol.wait (weights do not depend on the
//                 previous kernel).
//   warp 14       X producer: two 2-D SW128 tensor copies of the activation
//                 tile per k-block into the X ring (after griddepcontrol.wait).
//   warp 1        MMA issuer (+ TMEM allocation, 512 columns): one barrier
//                 wait per k-block (afull: the dequant warps publish the A
//                 slot only once the k-block's activation tile has landed
//                 too), 8 x tcgen05.mma.kind::i8 (K = 32 each), A from TMEM,
//                 B from the X ring; tcgen05.commit frees the X slot and the
//                 TMEM A slot and signals the epilogue at the end of a tile
//                 segment.
//   warps 2-9     two dequant warpgroups (the paper's ImFP compute WGs,
//                 P:415-416) taking alternate k-blocks: LDS of the packed
//                 codes and group parameters (one 2..16-byte LDS per k-block
//                 for the parameters), W slot released as soon as the codes
//                 are in registers, LiquidQuant (q*s + a) ^ 0x80 on four byte
//                 lanes per IMAD (packed.cpp:40-61), tcgen05.st of
//                 the INT8 result into the TMEM A ring (thread = weight row =
//                 TMEM lane).
//   warps 10-13   epilogue: tcgen05.ld of the INT32 accumulators, fused
//                 per-channel x per-token scaling and F32/F16/BF16 cast,
//                 stores (or the INT32 accumulators themselves), split-K
//                 exchange.
// The W ring (freed by the dequant warps) and the X ring (freed by the MMA)
// are separate, so a weight chunk's SMEM slot turns over after load latency +
// dequant only, and the weight stream keeps many chunks in flight whatever
// the token tile. All hand-offs are mbarrier arrivals (TMA complete_tx,
// tcgen05.commit, thread arrives); there is no __syncthreads in the mainloop.
//
// TMEM (512 columns): [0, acc_stages*acc_stride) INT32 accumulators, then
// the A ring of a_slots x 64 columns (one 256-wide k-block of int8 per slot).
//
// Work split: whole-tile rounds, then stream-K over the remaining tiles'
// (tile, k-block) space. A tile whose k-range spans several CTAs is reduced
// exactly in INT32 through a workspace (see the epilogue) -- or, in quad mode
// (two CTA pairs per tile in one 4-CTA cluster), by one DSMEM bulk copy from
// the contributor pair's shared memory into the finisher pair's; integer
// addition is associative, so results are bit-identical to the reference's
// fixed-order sum in any arrival order.
//
// CTA pairs (kPair): cluster rank bit 0 is the position in the pair (0 =
// leader, which issues the cta_group::2 MMAs), bit 1 (quad mode) the half of
// the tile's k-range.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "lqg_layout.h"
#include "sm100_ptx.cuh"

namespace lqg {

enum OutKind : uint32_t { kOutAcc = 0, kOutF32 = 1, kOutF16 = 2, kOutBF16 = 3 };

constexpr uint32_t kWarpW = 0;         // weight producer
constexpr uint32_t kWarpMMA = 1;       // MMA issuer, TMEM allocator
constexpr uint32_t kDequantWarp0 = 2;  // two warpgroups: warps 2-5, 6-9
constexpr uint32_t kDQWarps = 8;
constexpr uint32_t kEpiWarp0 = 10;     // warps 10-13
constexpr uint32_t kWarpX = 14;        // activation producer
constexpr uint32_t kThreads = 15 * 32;
constexpr uint32_t kMaxStages = 16;    // per ring
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

// Double-buffered accumulators whenever two fit next to an A ring of >= 2
// slots. The A ring may have an odd size although the two dequant
// warpgroups take alternate k-blocks: a warpgroup's ring position advances
// two slots per k-block and flips its parity on every wrap, i.e. parity =
// (k-block / slots) & 1; the empty barrier of k-block i's slot completes
// with the MMA of k-block i - slots, and MMAs complete in order, so when
// the warpgroup waits for it, the MMA of k-block i - 2 - slots (its previous
// wait) and hence of i - 2 * slots are done: the barrier is never two phases
// behind. (The W and X rings have no such order between the two warpgroups'
// TMA completions and stay even, see launch_core.)
__host__ __device__ inline TmemPlan tmem_plan(uint32_t BN, uint32_t max_acc_stages = 2) {
    constexpr uint32_t cols = 512;
    TmemPlan t;
    t.acc_stride = (BN + 31) / 32 * 32;
    t.acc_stages = (max_acc_stages >= 2 && 2 * t.acc_stride + 2 * kACols <= cols) ? 2u : 1u;
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
    int32_t* parts;            // split-K partials: per CTA kSlotCellsK int32 cells
    uint32_t* flags;           // per CTA: 1 = partial published (release), reset by the finisher
    uint32_t N;                // weight rows
    uint32_t KB, NT, MT;       // k-blocks, weight tiles, token tiles (of the largest group)
    uint32_t BN;               // tokens per tile (16..256, multiple of 16)
    uint32_t P;                // group params per k-block (1, 2, 4, 8)
    uint32_t chunk_bytes;      // bytes per (tile, k-block) weight chunk
    uint32_t out_kind;         // OutKind
    uint32_t x_stages;         // X ring depth
    uint32_t x_slot_bytes;     // bytes per X slot (this CTA's share of the activation tile)
    uint32_t w_stages;         // W ring depth (even)
    uint32_t w_base;           // byte offset of the W ring (after the X ring)
    uint32_t dp_rounds;        // whole tiles per CTA before the stream-K tail
    uint32_t raster_gm;        // token tiles per raster group
    uint32_t trace_slot;       // LQG_TRACE builds: launch index % 8
    uint32_t pair;             // 1: CTA pairs (cluster of 2, tcgen05 cta_group::2, M = 256):
                               //    NT/tiles count pair tiles, each CTA owns weight tile 2*nt+rank
                               //    and loads half of every activation tile
    uint32_t tiles;            // weight-tile x token-tile pairs (summed over groups)
    uint32_t sk_q, sk_r;       // stream-K iterations (tiles after the DP rounds x KB) = sk_q * units + sk_r
    uint32_t acc_stages;       // at most this many accumulator stages in TMEM (1 or 2; see tmem_plan)
    uint32_t quad;             // 1: clusters of 4 = the two CTA pairs of one split tile (units = 2 x tiles,
                               //    pair mode): the partial moves through DSMEM, not L2 (see the epilogue)
};

// Shared memory after the rings and barriers: TMEM address holder, then the
// token scales of the current tile (double).
constexpr uint32_t kMiscTsOff = 128;
constexpr uint32_t kMiscBytes = kMiscTsOff + kMaxBN * 8;
constexpr uint32_t kNumBarriers = 4 * kMaxStages + 3 * kMaxASlots + 9;

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

// First stream-K iteration of unit c: floor(total * c / G) with total =
// q * G + r (q, r from the host), in 32-bit arithmetic: q * c + r * c / G
// (r * c < G^2). A 64-bit division is a ~300-cycle subroutine on the GPU and
// sits on every CTA's prologue.
__device__ __forceinline__ uint32_t range_begin(uint32_t c, uint32_t G, uint32_t q, uint32_t r) {
    return q * c + (r * c) / G;
}

// CTAs whose range starts strictly inside tile `tile` (its contributors):
// [c_first, c_end). Each contributor's first segment is a piece of the tile.
__device__ __forceinline__ void split_contributors(uint32_t tile, uint32_t KB, uint32_t G, uint32_t q,
                                                   uint32_t r, uint32_t& c_first, uint32_t& c_end) {
    const uint32_t t0 = tile * KB, t1 = t0 + KB;
    const uint32_t total = q * G + r;
    uint32_t c = min(G, static_cast<uint32_t>(float(t0) * float(G) / float(total)));
    while (c > 0 && range_begin(c, G, q, r) > t0) --c;
    while (c < G && range_begin(c, G, q, r) <= t0) ++c;
    c_first = c;
    while (c < G && range_begin(c, G, q, r) < t1) ++c;
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
    uint32_t sk_tile0, sk_beg, sk_end;  // 32-bit: host guarantees total_iters * G < 2^32
    uint32_t sk_tile, sk_kb;            // first stream-K (tile, k-block) of this CTA
    uint32_t n_local;
};

// Scheduling units: CTAs, or CTA pairs (p.pair).
__device__ __forceinline__ uint32_t sched_units(const GemmParams& p) {
    return p.pair ? gridDim.x >> 1 : gridDim.x;
}
// Computed once per CTA (thread 0) and shared through SMEM.
__device__ __forceinline__ Sched make_sched(const GemmParams& p) {
    Sched s;
    const uint32_t G = sched_units(p);
    s.c = p.pair ? blockIdx.x >> 1 : blockIdx.x;
    s.dp_rounds = p.dp_rounds;
    s.sk_tile0 = s.dp_rounds * G;
    s.sk_beg = range_begin(s.c, G, p.sk_q, p.sk_r);
    s.sk_end = range_begin(s.c + 1, G, p.sk_q, p.sk_r);
    s.sk_tile = s.sk_tile0 + s.sk_beg / p.KB;
    s.sk_kb = s.sk_beg % p.KB;
    s.n_local = s.dp_rounds * p.KB + (s.sk_end - s.sk_beg);
    return s;
}

// Position in one CTA's iteration sequence (DP tiles, then its stream-K range).
// Self-contained (KB / dp_rounds come from the kernel parameter bank) so that
// no per-CTA schedule state stays live across the role loops.
struct Walk {
    uint32_t tile, kb, r, sk_tile, sk_kb;
    __device__ __forceinline__ void init(const Sched& s) {
        r = 0;
        sk_tile = s.sk_tile;
        sk_kb = s.sk_kb;
        if (s.dp_rounds > 0) {
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
        if (r < p.dp_rounds) {
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
    __device__ __forceinline__ bool in_dp(const GemmParams& p) const { return r < p.dp_rounds; }
};

// Ring position (slot, phase parity) advancing by `step` slots per use.
struct RingPos {
    uint32_t s, ph;
    __device__ __forceinline__ void adv(uint32_t step, uint32_t n) {
        s += step;
        if (s >= n) {
            s -= n;
            ph ^= 1;
        }
    }
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
    r.nt = p.pair ? 2 * nt + (ptx::cluster_ctarank() & 1u) : nt;
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

// Final reduction of a split large-token tile: for chunks ch0, ch0+step, ...
// the finisher's accumulator (TMEM) plus the nb gathered contributor
// partials (shared memory, [contributor][chunk][quad][row] int4 cells), then
// the scaled, cast output. Runs on the epilogue warps and, for the last batch,
// on the idle dequant warps too (the team finish, see the dequant role).
template <uint32_t kKind, bool kFan>
__device__ __forceinline__ void finish_chunks(const GemmParams& p, uint32_t ch0, uint32_t step, uint32_t nchunks,
                                              uint32_t acc_taddr, const int4* parts_smem, uint32_t nb,
                                              uint32_t part_bytes, uint32_t row, uint32_t n, uint32_t m0,
                                              uint32_t mlim, double cs, const double* ts_s) {
    for (uint32_t ch = ch0; ch < nchunks; ch += step) {
        uint32_t v[16];
        ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
        ptx::tmem_ld_wait();
        int32_t sum[16];
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j) sum[j] = int32_t(v[j]);
        for (uint32_t b = 0; b < nb; ++b) {
            const int4* scell = parts_smem + b * (part_bytes / 16) + ch * 4 * kTileN + row;
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q) {
                const int4 x = scell[q * kTileN];
                sum[4 * q] += x.x;
                sum[4 * q + 1] += x.y;
                sum[4 * q + 2] += x.z;
                sum[4 * q + 3] += x.w;
            }
        }
        if (n < p.N) store_chunk_k<kKind, kFan>(p, m0 + ch * 16, mlim, n, sum, cs, ts_s + ch * 16);
    }
}

// Team work of the CTA's last segment (tiles of more than kSentinelMaxChunks
// token chunks), from the schedule alone so that the dequant warps agree with
// the epilogue warps: kTeamFinish = the head piece of a split tile (flag +
// gather finisher). Measured and not done: a team publish of last-segment
// contributor pieces (1-2 % slower) and team stores of a last whole tile
// (neutral).
enum TeamRole : uint32_t { kTeamNone = 0, kTeamFinish = 1, kTeamWhole = 2 };

__device__ __forceinline__ uint32_t last_team_role(const GemmParams& p, uint32_t dp_rounds, uint32_t sk_beg,
                                                   uint32_t sk_end) {
    if (p.BN / 16 <= kSentinelMaxChunks) return kTeamNone;
    if (sk_end == sk_beg) return dp_rounds ? kTeamWhole : kTeamNone;
    const uint32_t last_tile = (sk_end - 1) / p.KB;  // relative to the stream-K tiles
    const uint32_t seg_beg = max(sk_beg, last_tile * p.KB);
    if (seg_beg > last_tile * p.KB) return kTeamNone;
    return sk_end - seg_beg < p.KB ? kTeamFinish : kTeamWhole;
}

// Named barrier 1 of the 4 epilogue warps (bar.sync is warp-aligned: the warp
// reconverges first, as the mbarrier try_wait loops before it are invisible
// to the compiler's reconvergence analysis).
__device__ __forceinline__ void epi_bar() {
    __syncwarp();
    asm volatile("bar.sync 1, 128;" ::: "memory");
}

#ifdef LQG_TRACE_KB
// Debug builds: per-k-block %globaltimer events (ns) of CTAs 0 and 1 (k-blocks 0..63):
// 0 W issued, 1 X issued, 2 dequant W ready, 3 dequant A slot free,
// 4 dequant A published, 5 MMA A ready, 6 MMA issued.
__device__ long long g_lqg_kb[2 * 64 * 8];  // CTAs 0 and 1 (a pair's leader and peer)
#define LQG_KB(i, e)                                                                                   \
    do {                                                                                               \
        if (blockIdx.x < 2 && (i) < 64) {                                                              \
            long long t_;                                                                              \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)::"memory");                           \
            g_lqg_kb[(blockIdx.x * 64 + (i)) * 8 + (e)] = t_;                                          \
        }                                                                                              \
    } while (0)
#else
#define LQG_KB(i, e) ((void)0)
#endif

#ifdef LQG_TRACE_SEG
// Debug builds: per-segment (accumulator stage use) %globaltimer events of CTAs
// 0..7, segments 0..31: 0 MMA starts waiting for the stage, 1 stage free,
// 2 last MMA of the segment issued, 3 epilogue sees the accumulator, 4 stage
// released, 5 epilogue segment done, 6 k-blocks in the segment, 7 kind (0 whole
// tile, 1 contributor, 2 finisher), 8 / 9 whole tile: epilogue warp 10's
// cycles in TMEM load + wait / in scale + store.
__device__ long long g_lqg_seg[8 * 32 * 16];
#define LQG_SEG(j, e, v)                                                                        \
    do {                                                                                        \
        if (blockIdx.x < 8 && (j) < 32) g_lqg_seg[(blockIdx.x * 32 + (j)) * 16 + (e)] = (v);   \
    } while (0)
#define LQG_SEGT(j, e)                                                          \
    do {                                                                        \
        long long t_;                                                           \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)::"memory");        \
        LQG_SEG(j, e, t_);                                                      \
    } while (0)
#else
#define LQG_SEG(j, e, v) ((void)0)
#define LQG_SEGT(j, e) ((void)0)
#endif

#ifdef LQG_TRACE
// Debug builds: per-CTA %globaltimer events and per-role wait cycles.
__device__ unsigned long long g_lqg_trace[8 * 160 * 16];
__device__ __forceinline__ void trace(uint32_t slot, uint32_t e) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    g_lqg_trace[(slot * 160 + blockIdx.x) * 16 + e] = t;
}
#define LQG_T(e) trace(p.trace_slot, e)
#define LQG_TV(e, v) (g_lqg_trace[(p.trace_slot * 160 + blockIdx.x) * 16 + (e)] = (v))
#define LQG_WAIT(acc_, call_)                  \
    do {                                       \
        const long long t0_ = clock64();       \
        call_;                                 \
        acc_ += clock64() - t0_;               \
    } while (0)
#else
#define LQG_T(e) ((void)0)
#define LQG_TV(e, v) ((void)0)
#define LQG_WAIT(acc_, call_) call_
#endif

template <uint32_t V>
struct UConst {
    static constexpr uint32_t value = V;
};

// kG > 1: grouped launch over up to kG weight groups (MoE experts).
// kFan: the epilogue also stores every tile into p.fan[0..n_fan) (fused
// all-gather of the N-split driver); a separate instantiation so the plain
// kernel's epilogue is untouched.
// kPair: CTA pairs (cluster of two, tcgen05 cta_group::2, M = 256): each
// CTA dequantizes its own 128 weight rows into its TMEM and loads half of the
// activation tile (N/2 tokens); the leader issues one M=256 MMA that reads the
// B halves from both CTAs' shared memory, which halves the activation
// shared-memory traffic per SM.
template <uint32_t kKind, uint32_t kG, bool kFan, bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
    lqg_w4a8_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const GemmParams p,
                         const __grid_constant__ GroupTable<kG> gt) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the SW128 activation tiles.
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t pad = (1024 - (raw_addr & 1023)) & 1023;
    uint8_t* smem = smem_raw + pad;
    const uint32_t smem_base = raw_addr + pad;

    const uint32_t SX = p.x_stages, SW = p.w_stages;
    const uint32_t ring_bytes = p.w_base + SW * p.chunk_bytes;  // X ring, then W ring
    const uint32_t bar_base = smem_base + ((ring_bytes + 7) & ~7u);
    auto wfull_bar = [&](uint32_t s) { return bar_base + 8 * s; };
    auto wempty_bar = [&](uint32_t s) { return bar_base + 8 * (kMaxStages + s); };
    auto xfull_bar = [&](uint32_t s) { return bar_base + 8 * (2 * kMaxStages + s); };
    auto xempty_bar = [&](uint32_t s) { return bar_base + 8 * (3 * kMaxStages + s); };
    constexpr uint32_t kB = 4 * kMaxStages;
    auto afull_bar = [&](uint32_t a) { return bar_base + 8 * (kB + a); };
    auto aempty_bar = [&](uint32_t a) { return bar_base + 8 * (kB + kMaxASlots + a); };
    auto accfull_bar = [&](uint32_t a) { return bar_base + 8 * (kB + 2 * kMaxASlots + a); };
    auto accempty_bar = [&](uint32_t a) { return bar_base + 8 * (kB + 2 * kMaxASlots + 2 + a); };
    const uint32_t fin_bar = bar_base + 8 * (kB + 2 * kMaxASlots + 4);  // split-K gather (finisher)
    // team finish hand-over: epilogue -> dequant warps (tile gathered), and back
    const uint32_t team_ready = bar_base + 8 * (kB + 2 * kMaxASlots + 5);
    const uint32_t team_done = bar_base + 8 * (kB + 2 * kMaxASlots + 6);
    // first half of an A slot (K columns 0..127) read: the MMA warp commits after
    // the k-block's first four MMAs
    auto aempty_lo_bar = [&](uint32_t a) { return bar_base + 8 * (kB + 2 * kMaxASlots + 7 + a); };
    // every dequant warp has finished reading the W ring (the finisher's
    // gather reuses the rings; the order also runs through the MMA, this
    // makes it explicit)
    const uint32_t dq_done = bar_base + 8 * (kB + 3 * kMaxASlots + 7);
    // quad mode: the finisher's ring is free and its fin_bar armed (remote arrive)
    const uint32_t qready = bar_base + 8 * (kB + 3 * kMaxASlots + 8);
    uint8_t* misc = smem + ((ring_bytes + 7) & ~7u) + 8 * (kB + 3 * kMaxASlots + 9);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(misc);
    double* ts_s = reinterpret_cast<double*>(misc + kMiscTsOff);  // kMaxBN token scales, as double
    uint32_t* team_info = reinterpret_cast<uint32_t*>(misc + 64);  // team finish: tile, acc column, nb

    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t G = sched_units(p);
    const uint32_t KB = p.KB;
    constexpr uint32_t kTmemCols = 512;
    const TmemPlan tp = tmem_plan(p.BN, p.acc_stages);
    // cluster = one CTA pair, or (p.quad) the two pairs of one split tile
    const uint32_t crank = kPair ? ptx::cluster_ctarank() : 0u;
    const uint32_t rank = crank & 1u;   // 0 = pair leader
    const uint32_t lead = crank & ~1u;  // the pair leader's cluster rank
    // barriers the pair leader waits on, as seen from this CTA
    auto leader = [&](uint32_t bar) { return kPair ? ptx::mapa(bar, lead) : bar; };

    if (threadIdx.x == 0) LQG_T(0);
    if (warp == 0) {
        // barrier init spread over the lanes of warp 0 (one mbarrier per lane-step)
        for (uint32_t s = lane; s < SW; s += 32) {
            ptx::mbar_init(wfull_bar(s), 1);
            ptx::mbar_init(wempty_bar(s), 4);  // the 4 warps of the dequant WG of this k-block
        }
        for (uint32_t s = lane; s < SX; s += 32) {
            ptx::mbar_init(xfull_bar(s), 1);
            ptx::mbar_init(xempty_bar(s), 1);
        }
        if (lane < kMaxASlots) {
            ptx::mbar_init(afull_bar(lane), kPair ? 8 : 4);  // the dequant WG's warps (of both CTAs)
            ptx::mbar_init(aempty_bar(lane), 1);
            ptx::mbar_init(aempty_lo_bar(lane), 1);
        }
        if (lane < 2) {
            ptx::mbar_init(accfull_bar(lane), 1);
            ptx::mbar_init(accempty_bar(lane), kPair ? 8 : 4);  // one arrive per epilogue warp
        }
        if (lane == 0) {
            ptx::mbar_init(fin_bar, 1);
            ptx::mbar_init(team_ready, 1);         // the epilogue's leading thread
            ptx::mbar_init(team_done, kDQWarps);   // one arrive per dequant warp
            ptx::mbar_init(dq_done, kDQWarps);
            ptx::mbar_init(qready, 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == kWarpX && lane == 0) ptx::prefetch_tmap(&tmap_x);
    if (warp == kWarpMMA) {
        if (kPair)
            ptx::tmem_alloc_pair(ptx::smem_u32(tmem_holder), kTmemCols);
        else
            ptx::tmem_alloc(ptx::smem_u32(tmem_holder), kTmemCols);
    }
    ptx::tc_fence_before();
    __syncthreads();
#ifdef LQG_TRACE_PRO
    if (threadIdx.x == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        LQG_TV(3, smid);
    }
#endif
    if (kPair) ptx::cluster_sync();  // the peer's barriers are initialised before any remote arrive
    ptx::tc_fence_after();
    // The CTA owns the SM's whole TMEM (512 columns, one CTA per SM), so the
    // allocation always starts at lane 0 / column 0: TMEM addresses below are
    // compile-time offsets (kept in uniform registers by the MMA warp).
    if (*tmem_holder != 0) __trap();
    constexpr uint32_t tmem_base = 0;
    // The schedule is recomputed by every thread from kernel parameters and
    // the block index (warp-uniform values, no shared-memory round trip).
    const Sched sch = make_sched(p);
    const uint32_t n_local = sch.n_local;
    // PDL: the next kernel in the stream may launch now; its CTAs only
    // prefetch weights until their griddepcontrol.wait, which returns once
    // this grid has completed and its memory is visible. Everything below
    // that reads or writes dependent memory (activations, token scales,
    // outputs, workspace) sits behind griddepcontrol.wait here too. (Issued
    // after the barrier above: the issuing warp stops counting towards CTA
    // barriers.)
    if (threadIdx.x == 0) ptx::launch_dependents();
    if (threadIdx.x == 0) LQG_T(1);

    if (warp == kWarpW) {
        // ------------------------------------------------------------ W producer
        // A single-pass weight stream is EVICT_FIRST; weights re-read by
        // several token tiles EVICT_LAST.
        const uint64_t pol_w = p.MT == 1 ? ptx::policy_evict_first() : ptx::policy_evict_last();
        Walk ww;
        ww.init(sch);
        auto chunk_src = [&](uint32_t tile, uint32_t kb) {
            const TileRef r = tile_ref(tile, p, gt);
            return r.wimg + (uint64_t(r.nt) * KB + kb) * p.chunk_bytes;
        };
        const uint8_t* src = chunk_src(ww.tile, ww.kb);
        RingPos w{0, 0};
        for (uint32_t i = 0; i < n_local; ++i) {
            ptx::mbar_wait(wempty_bar(w.s), w.ph ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(wfull_bar(w.s), p.chunk_bytes);
                ptx::bulk_g2s(smem_base + p.w_base + w.s * p.chunk_bytes, src, p.chunk_bytes, wfull_bar(w.s), pol_w);
                LQG_KB(i, 0);
            }
            __syncwarp();
            if (ww.next(p))
                src = chunk_src(ww.tile, ww.kb);
            else
                src += p.chunk_bytes;
            w.adv(1, SW);
        }
    } else if (warp == kWarpX) {
        // ------------------------------------------------------------ X producer
        const uint64_t pol_x = ptx::policy_evict_last();
        const uint32_t atom_bytes = (kPair ? p.BN / 2 : p.BN) * kXAtom;
        Walk xw;
        xw.init(sch);
        uint32_t xrow0 = tile_ref(xw.tile, p, gt).row0;
        ptx::griddep_wait();
        if (lane == 0) LQG_T(2);
        RingPos x{0, 0};
        for (uint32_t i = 0; i < n_local; ++i) {
            ptx::mbar_wait(xempty_bar(x.s), x.ph ^ 1);
            if (ptx::elect_one()) {
                const uint32_t slot = smem_base + x.s * p.x_slot_bytes;
                const int32_t k0 = int32_t(xw.kb * kKBlock);
                if (kPair) {
                    // both halves count on the leader's barrier; the leader expects the whole tile
                    if (rank == 0) ptx::mbar_arrive_expect_tx(xfull_bar(x.s), 2 * p.x_slot_bytes);
                    const int32_t m0 = int32_t(xrow0 + rank * (p.BN / 2));
                    const uint32_t fb = ptx::mapa(xfull_bar(x.s), lead);
                    ptx::tma_2d_g2s_pair(slot, &tmap_x, k0, m0, fb, pol_x);
                    ptx::tma_2d_g2s_pair(slot + atom_bytes, &tmap_x, k0 + int32_t(kXAtom), m0, fb, pol_x);
                } else {
                    ptx::mbar_arrive_expect_tx(xfull_bar(x.s), p.x_slot_bytes);
                    const int32_t m0 = int32_t(xrow0);
                    ptx::tma_2d_g2s(slot, &tmap_x, k0, m0, xfull_bar(x.s), pol_x);
                    ptx::tma_2d_g2s(slot + atom_bytes, &tmap_x, k0 + int32_t(kXAtom), m0, xfull_bar(x.s), pol_x);
                }
                LQG_KB(i, 1);
            }
            __syncwarp();
            if (xw.next(p)) xrow0 = tile_ref(xw.tile, p, gt).row0;
            x.adv(1, SX);
        }
    } else if (warp == kWarpMMA && (!kPair || rank == 0)) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = ptx::idesc_i8(kPair ? 2 * kTileN : kTileN, p.BN);
        const uint64_t desc0 = ptx::sw128_kmajor_desc(smem_base);
        const uint32_t slot_desc = p.x_slot_bytes >> 4;
        const uint32_t atom_desc = ((kPair ? p.BN / 2 : p.BN) * kXAtom) >> 4;
        // Segment lengths (k-blocks accumulated into one accumulator stage):
        // dp_rounds whole tiles, then the stream-K range's first (partial)
        // tile, then whole tiles, the last one possibly cut by the range end.
        const uint32_t dp_iters = sch.dp_rounds * KB;
        auto seg_len = [&](uint32_t i) -> uint32_t {
            if (i < dp_iters) return KB;
            return min(i == dp_iters ? KB - sch.sk_kb : KB, n_local - i);
        };
        uint32_t seg_left = n_local ? seg_len(0) : 0;
        bool seg_start = true;
        RingPos x{0, 0}, a{0, 0};
        uint32_t as = 0, acc_ph = 0;
#ifdef LQG_TRACE_SEG
        uint32_t sidx = 0;
#endif
#ifdef LQG_TRACE
        long long w_acc = 0, w_a = 0, w_x = 0, w_issue = 0;  // w_x: unused (X folded into afull)
        const long long t_mma0 = clock64();
#endif
        auto wait_ready = [&]() {
            if (seg_start) {
                if (lane == 0) LQG_SEGT(sidx, 0);
                LQG_WAIT(w_acc, ptx::mbar_wait(accempty_bar(as), acc_ph ^ 1));
                if (lane == 0) LQG_SEGT(sidx, 1);
            }
            LQG_WAIT(w_a, ptx::mbar_wait(afull_bar(a.s), a.ph));
            ptx::tc_fence_after();
        };
        auto mma = [&](uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t k8, bool first) {
            const uint64_t bd = bdesc + (k8 / 4) * atom_desc + (k8 % 4) * 2;
            if (kPair)
                ptx::mma_i8_ts_pair(d_tmem, a_tmem + k8 * 8, bd, idesc, first ? 0u : 1u);
            else
                ptx::mma_i8_ts(d_tmem, a_tmem + k8 * 8, bd, idesc, first ? 0u : 1u);
        };
        auto commit = [&](uint32_t bar) {
            if (kPair)
                ptx::mma_commit_pair(bar, uint16_t(3u << lead));
            else
                ptx::mma_commit(bar);
        };
        for (uint32_t i = 0; i < n_local; ++i) {
            wait_ready();
            if (lane == 0) LQG_KB(i, 5);
            if (i == 0 && lane == 0) LQG_T(4);
            if (i + 1 == n_local && lane == 0) LQG_T(5);
            const bool seg_end = seg_left == 1;
#ifdef LQG_TRACE
            const long long t_is0 = clock64();
#endif
            if (ptx::elect_one()) {
                const uint32_t d_tmem = tmem_base + as * tp.acc_stride;
                const uint32_t a_tmem = tmem_base + tp.a_base + a.s * kACols;
                const uint64_t bdesc = desc0 + uint64_t(x.s * slot_desc);
                // The first half of the A slot is free once the first four
                // MMAs have read it: its own commit lets the dequant warps
                // refill that half while the second half is still being read.
#pragma unroll
                for (uint32_t k8 = 0; k8 < kSubBlocks / 2; ++k8) mma(d_tmem, a_tmem, bdesc, k8, seg_start && k8 == 0);
                commit(aempty_lo_bar(a.s));
#pragma unroll
                for (uint32_t k8 = kSubBlocks / 2; k8 < kSubBlocks; ++k8) mma(d_tmem, a_tmem, bdesc, k8, false);
                commit(xempty_bar(x.s));
                commit(aempty_bar(a.s));
                if (seg_end) commit(accfull_bar(as));
                if (seg_end) LQG_SEGT(sidx, 2);
                LQG_KB(i, 6);
            }
            __syncwarp();
#ifdef LQG_TRACE
            w_issue += clock64() - t_is0;
#endif
#ifdef LQG_TRACE_SEG
            if (seg_end) ++sidx;
#endif
            if (seg_end && ++as == tp.acc_stages) {
                as = 0;
                acc_ph ^= 1;
            }
            seg_start = seg_end;
            if (--seg_left == 0 && i + 1 < n_local) seg_left = seg_len(i + 1);
            x.adv(1, SX);
            a.adv(1, tp.a_slots);
        }
#ifdef LQG_TRACE
#ifndef LQG_TRACE_PRO
        if (lane == 0) {  // MMA-warp wait cycles: accumulator, A operand, activation tile, total
            LQG_TV(12, (unsigned long long)w_acc);
            LQG_TV(13, (unsigned long long)w_a);
            LQG_TV(14, (unsigned long long)w_x);
            LQG_TV(15, (unsigned long long)(clock64() - t_mma0));
            LQG_TV(3, (unsigned long long)w_issue);
        }
#endif
#endif
    } else if (warp >= kDequantWarp0 && warp < kEpiWarp0) {
        // ------------------------------------------------------------ dequant WGs
        // WG w dequantizes the whole k-blocks w, w+2, w+4, ... of this CTA.
        // Both rings are even, so WG w always uses the same half of the W
        // slots and A slots and observes every phase of each (a parity wait
        // can never alias an older phase).
        const uint32_t wg = (warp - kDequantWarp0) / 4;
        const uint32_t sp = warp % 4;         // TMEM sub-partition
        const uint32_t row = sp * 32 + lane;  // weight row within the tile = TMEM lane
        const uint32_t a_lane = tmem_base + ((sp * 32) << 16) + tp.a_base;
        const uint8_t* wring = smem + p.w_base;
        auto run = [&](auto kp) {
            constexpr uint32_t P = decltype(kp)::value;
            constexpr uint32_t kSubPerP = kSubBlocks / P;
#ifdef LQG_TRACE
            long long dq_w = 0, dq_a = 0;
            const long long t_dq0 = clock64();
#endif
            RingPos w{wg, 0}, a{wg, 0}, xr{wg, 0};
            // The activation tile of this k-block must have landed before the
            // A operand is published: the MMA warp then waits on a single
            // barrier (afull) per k-block. In a pair the leader's barrier
            // counts both CTAs' halves, so only the leader's warps wait.
            auto wait_x = [&]() {
                if (!kPair || rank == 0) ptx::mbar_wait(xfull_bar(xr.s), xr.ph);
                xr.adv(2, SX);
            };
            for (uint32_t i = wg; i < n_local; i += 2) {
                LQG_WAIT(dq_w, ptx::mbar_wait(wfull_bar(w.s), w.ph));
                if (warp % 4 == 2 && lane == 0) LQG_KB(i, 2);
                const uint8_t* wchunk = wring + w.s * p.chunk_bytes;
                // all P group parameters of this row: one 2..16-byte LDS
                uint32_t prm[(P + 1) / 2];
                const uint8_t* pa = wchunk + kCodeBytes + row * (2 * P);
                if constexpr (P == 1) {
                    prm[0] = *reinterpret_cast<const uint16_t*>(pa);
                } else if constexpr (P == 2) {
                    prm[0] = *reinterpret_cast<const uint32_t*>(pa);
                } else if constexpr (P == 4) {
                    const uint2 t = *reinterpret_cast<const uint2*>(pa);
                    prm[0] = t.x;
                    prm[1] = t.y;
                } else {
                    const uint4 t = *reinterpret_cast<const uint4*>(pa);
                    prm[0] = t.x;
                    prm[1] = t.y;
                    prm[2] = t.z;
                    prm[3] = t.w;
                }
                const uint32_t a_taddr = a_lane + a.s * kACols;
                auto dq_param = [&](uint32_t c, uint32_t& sc, uint32_t& a4) {
                    const uint32_t pi = c / kSubPerP;  // parameter region of sub-block c
                    const uint32_t sa = (prm[pi / 2] >> (16 * (pi % 2))) & 0xFFFFu;
                    sc = sa & 0xFFu;
                    a4 = (sa >> 8) * 0x01010101u;
                };
                uint4 v[kSubBlocks];
#pragma unroll
                for (uint32_t c = 0; c < kSubBlocks; ++c)
                    v[c] = *reinterpret_cast<const uint4*>(wchunk + (c * kTileN + row) * 16);
                // The whole k-block is converted before the A slot is claimed, so
                // once the MMA frees the slot only the two TMEM stores stand
                // between it and the next afull arrival (two A slots per
                // warpgroup at the largest token tile: this latency, not the
                // ALU work, gates the tensor pipe).
                uint32_t o[2][32];
#pragma unroll
                for (uint32_t c = 0; c < kSubBlocks; ++c) {
                    uint32_t sc, a4;
                    dq_param(c, sc, a4);
                    uint32_t* oc = &o[c / 4][8 * (c % 4)];
                    lqq_dequant_word(v[c].x, sc, a4, oc[0], oc[1]);
                    lqq_dequant_word(v[c].y, sc, a4, oc[2], oc[3]);
                    lqq_dequant_word(v[c].z, sc, a4, oc[4], oc[5]);
                    lqq_dequant_word(v[c].w, sc, a4, oc[6], oc[7]);
                }
                // every code of the chunk has been consumed: free the W slot
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(wempty_bar(w.s));
                // Half by half: the first half of the slot is rewritten as soon
                // as the previous k-block's first four MMAs have read it.
                LQG_WAIT(dq_a, ptx::mbar_wait(aempty_lo_bar(a.s), a.ph ^ 1));
                if (warp % 4 == 2 && lane == 0) LQG_KB(i, 3);
                ptx::tc_fence_after();
                ptx::tmem_st_x32(a_taddr, o[0]);
                ptx::mbar_wait(aempty_bar(a.s), a.ph ^ 1);
                ptx::tc_fence_after();
                ptx::tmem_st_x32(a_taddr + 32, o[1]);
                ptx::tmem_st_wait();
                if (warp % 4 == 2 && lane == 0) LQG_KB(i, 7);
                ptx::tc_fence_before();
                wait_x();
                __syncwarp();
                if (lane == 0) {
                    if (kPair && rank != 0)
                        ptx::mbar_arrive_cluster_relaxed(leader(afull_bar(a.s)));
                    else
                        ptx::mbar_arrive(afull_bar(a.s));
                    if (warp % 4 == 2) LQG_KB(i, 4);
                }
                w.adv(2, SW);
                a.adv(2, tp.a_slots);
            }
#if defined(LQG_TRACE) && !defined(LQG_TRACE_PRO)
            if (warp == kDequantWarp0 && lane == 0) {  // dequant waits: weights, A slot, total
                LQG_TV(11, (unsigned long long)(clock64() - t_dq0));
                LQG_TV(9, (unsigned long long)dq_w);
                LQG_TV(10, (unsigned long long)dq_a);
            }
#endif
        };
        switch (p.P) {
            case 1: run(UConst<1>{}); break;
            case 2: run(UConst<2>{}); break;
            case 4: run(UConst<4>{}); break;
            default: run(UConst<8>{}); break;
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(dq_done);
        // Team finish (see the epilogue's large finisher): the last batch's
        // reduction and stores of chunks 1 + wg, 4 + wg, ... of the
        // finisher tile, once the epilogue warps have gathered it.
        const uint32_t team = last_team_role(p, sch.dp_rounds, sch.sk_beg, sch.sk_end);
        if (team == kTeamFinish) {
            ptx::mbar_wait(team_ready, 0);
            ptx::tc_fence_after();
            const TileRef tr = tile_ref(team_info[0], p, gt);
            const uint32_t n = tr.nt * kTileN + row;
            const double cs = kKind != kOutAcc ? double(tr.cs[n]) : 0.0;
            const uint32_t acc_taddr = tmem_base + ((sp * 32) << 16) + team_info[1];
            finish_chunks<kKind, kFan>(p, 1 + wg, 3, p.BN / 16, acc_taddr, reinterpret_cast<const int4*>(smem),
                               team_info[2], p.BN * kTileN * 4, row, n, tr.row0, tr.mlim, cs, ts_s);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(team_done);
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ------------------------------------------------------------ epilogue
        const uint32_t sp = warp % 4;
        const uint32_t row = sp * 32 + lane;
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t et = threadIdx.x - kEpiWarp0 * 32;  // 0..127
        const uint32_t nchunks = p.BN / 16;
        constexpr bool scaled = kKind != kOutAcc;
        ptx::griddep_wait();
        uint32_t as = 0, acc_ph = 0, fin_ph = 0;
        uint32_t i = 0;
        Walk ew;
        ew.init(sch);
#ifdef LQG_TRACE_SEG
        uint32_t eidx = 0;
#endif
        auto release_acc = [&](uint32_t cur_as) {
            if (et == 0) LQG_SEGT(eidx, 4);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (kPair && rank != 0)
                    ptx::mbar_arrive_cluster_relaxed(leader(accempty_bar(cur_as)));
                else
                    ptx::mbar_arrive(accempty_bar(cur_as));
            }
        };
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
            // Split-K cells of up to kCB contributors for one 16-token chunk:
            // [contributor][quad]. Loaded one chunk ahead (software pipeline).
            constexpr uint32_t kCB = 4;  // contributors per L2 round trip
            int4 cb[kCB][4];
            auto cell_of = [&](uint32_t c, uint32_t ch) {
                const uint32_t cs_slot = kPair ? 2 * c + rank : c;  // the matching CTA of a contributor pair
                return reinterpret_cast<int4*>(p.parts + uint64_t(cs_slot) * kSlotCellsK + (small ? 0u : kSmallCells)) +
                       ch * 4 * kTileN + row;
            };
            auto load_batch = [&](uint32_t c, uint32_t ch) {
                const uint32_t nb = min(kCB, c_end - c);
#pragma unroll
                for (uint32_t b = 0; b < kCB; ++b)
                    if (b < nb)
#pragma unroll
                        for (uint32_t q = 0; q < 4; ++q) cb[b][q] = __ldcg(cell_of(c + b, ch) + q * kTileN);
            };
            if (finisher) {
                split_contributors(tile - sch.sk_tile0, KB, G, p.sk_q, p.sk_r, c_first, c_end);
                if (small) load_batch(c_first, 0);
            }
            epi_bar();
            ptx::mbar_wait_parked(accfull_bar(as), acc_ph);  // idle for a tile mainloop
            if (et == 0) {
                LQG_SEGT(eidx, 3);
                LQG_SEG(eidx, 6, n_iters);
                LQG_SEG(eidx, 7, n_iters == KB ? 0 : (kb0 > 0 ? 1 : 2));
            }
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
#ifdef LQG_TRACE_SEG
                long long c_ld = 0, c_st = 0;
#endif
                for (uint32_t ch = 0; ch < nchunks; ++ch) {
                    uint32_t v[16];
#ifdef LQG_TRACE_SEG
                    const long long c0 = clock64();
#endif
                    ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                    ptx::tmem_ld_wait();
#ifdef LQG_TRACE_SEG
                    const long long c1 = clock64();
                    c_ld += c1 - c0;
#endif
                    if (ch + 1 == nchunks) release_acc(cur_as);
                    if (n < p.N) {
                        int32_t a[16];
#pragma unroll
                        for (uint32_t j = 0; j < 16; ++j) a[j] = int32_t(v[j]);
                        store_chunk_k<kKind, kFan>(p, m0 + ch * 16, mlim, n, a, cs, ts_s + ch * 16);
                    }
#ifdef LQG_TRACE_SEG
                    asm volatile("" ::: "memory");
                    c_st += clock64() - c1;
#endif
                }
#ifdef LQG_TRACE_SEG
                if (et == 0) {
                    LQG_SEG(eidx, 8, c_ld);
                    LQG_SEG(eidx, 9, c_st);
                }
#endif
            } else if (kb0 > 0 && kPair && p.quad) {
                // Quad mode: this pair holds the second half of the tile's
                // k-range and the finisher pair is in the same cluster (ranks
                // crank - 2). This is the CTA's only segment, so its rings are
                // idle: stage the INT32 partial in shared memory ([chunk][quad]
                // [row] int4 cells, the finisher's layout) and move it with one
                // DSMEM bulk copy once the finisher's ring is free -- no L2
                // round trip, no fence, no flag.
                const uint32_t part_bytes = p.BN * kTileN * 4;
                if (et == 0) ptx::mbar_wait(dq_done, 0);  // the W ring's last reads are done
                epi_bar();
                int4* sm4w = reinterpret_cast<int4*>(smem);
                for (uint32_t ch = 0; ch < nchunks; ++ch) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                    ptx::tmem_ld_wait();
                    if (ch + 1 == nchunks) release_acc(cur_as);
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q)
                        sm4w[ch * 4 * kTileN + q * kTileN + row] =
                            make_int4(int32_t(v[4 * q]), int32_t(v[4 * q + 1]), int32_t(v[4 * q + 2]),
                                      int32_t(v[4 * q + 3]));
                }
                ptx::fence_proxy_async();  // the staged cells, for the bulk copy (async proxy)
                epi_bar();
                if (et == 0) {
                    ptx::mbar_wait(qready, 0);  // the finisher's ring is free, its fin_bar armed
                    ptx::bulk_s2s_cluster(ptx::mapa(smem_base, crank - 2), smem_base, part_bytes,
                                          ptx::mapa(fin_bar, crank - 2));
                    LQG_T(7);
                }
                // (the source cells stay valid until the copy completes: the
                // finisher reaches the closing cluster barrier only after it)
            } else if (kb0 > 0) {
                // Contributor piece of a split tile (always this CTA's first
                // segment): publish the INT32 partial into this CTA's cells.
                // Small tiles: no fence and no flag -- |partial| <= 133120 *
                // 127^2 < 2^31, so INT32_MIN never occurs as a value and marks
                // "not published"; each 16-byte cell is written by one st.cg
                // and re-read by the finisher until no lane holds the sentinel.
                // Large tiles: every cell, then a fence and a release flag per CTA.
                int32_t* slot = p.parts + uint64_t(blockIdx.x) * kSlotCellsK + (small ? 0u : kSmallCells);
                for (uint32_t ch = 0; ch < nchunks; ++ch) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(acc_taddr + ch * 16, v);
                    ptx::tmem_ld_wait();
                    if (ch + 1 == nchunks) release_acc(cur_as);
                    // [chunk][quad q][row] int4 cells: a warp's stores are 512
                    // contiguous bytes, and the finisher's bulk copy is one block
                    int4* cell = reinterpret_cast<int4*>(slot) + ch * 4 * kTileN + row;
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q)
                        __stcg(cell + q * kTileN, make_int4(int32_t(v[4 * q]), int32_t(v[4 * q + 1]),
                                                            int32_t(v[4 * q + 2]), int32_t(v[4 * q + 3])));
                }
                if (!small) {
                    // large tiles: every epilogue thread's stores, then one release flag
                    __threadfence();
                    epi_bar();
                    if (et == 0) ptx::st_release_u32(p.flags + blockIdx.x, 1u);
                }
                if (et == 0) LQG_T(7);
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
                        for (uint32_t c = c_first; c < c_end; c += kCB) {
                            const uint32_t nb = min(kCB, c_end - c);
                            if (c != c_first) load_batch(c, ch);
                            auto pend = [](const int4& x) {
                                return x.x == INT32_MIN || x.y == INT32_MIN || x.z == INT32_MIN ||
                                       x.w == INT32_MIN;
                            };
                            for (;;) {
                                uint32_t mask = 0;
#pragma unroll
                                for (uint32_t b = 0; b < kCB; ++b)
#pragma unroll
                                    for (uint32_t q = 0; q < 4; ++q)
                                        mask |= (b < nb && pend(cb[b][q])) ? (1u << (4 * b + q)) : 0u;
                                if (!mask) break;
                                __nanosleep(32);
#pragma unroll
                                for (uint32_t b = 0; b < kCB; ++b)
#pragma unroll
                                    for (uint32_t q = 0; q < 4; ++q)
                                        if (mask & (1u << (4 * b + q)))
                                            cb[b][q] = ptx::ld_relaxed_v4(cell_of(c + b, ch) + q * kTileN);
                            }
#pragma unroll
                            for (uint32_t b = 0; b < kCB; ++b) {
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
                            if (c + kCB >= c_end && ch + 1 < nchunks) load_batch(c_first, ch + 1);
                        }
                        if (n < p.N) store_chunk_k<kKind, kFan>(p, m0 + ch * 16, mlim, n, sum, cs, ts_s + ch * 16);
                    }
                } else {
                    // Large token tiles: this is the CTA's last segment, so the
                    // SMEM rings are idle. Wait (acquire) until every contributor
                    // has raised its flag, then gather the partials (one
                    // contiguous BN*512-byte block each) by TMA bulk copies, as
                    // many per batch as the rings hold, and sum them from SMEM:
                    // two L2 round trips per batch instead of one per 16-token
                    // chunk. Flags are reset for the next launch (which touches
                    // them only after griddepcontrol.wait).
                    const uint32_t part_bytes = p.BN * kTileN * 4;
                    const uint32_t nb_max = max(1u, ring_bytes / part_bytes);
                    const int4* sm4 = reinterpret_cast<const int4*>(smem);
#ifdef LQG_TRACE_PRO
                    if (et == 0) LQG_T(9);
#endif
#ifdef LQG_TRACE_PRO
                    if (et == 0) LQG_T(10);
#endif
                    for (uint32_t c0 = c_first;; c0 += nb_max) {
                        const uint32_t nb = min(nb_max, c_end - c0);
                        const bool last_batch = c0 + nb >= c_end;
                        if (kPair && p.quad && et == 0 && nb) {
                            // quad mode: the other half's pair (ranks crank + 2)
                            // copies its partial into this ring (DSMEM)
                            ptx::mbar_wait(dq_done, 0);  // the W ring's last reads are done
                            ptx::mbar_arrive_expect_tx(fin_bar, part_bytes);
                            ptx::fence_proxy_async();  // prior generic ring reads vs the async-proxy writes
                            ptx::mbar_arrive_cluster(ptx::mapa(qready, crank + 2));
                        } else if (et == 0 && nb) {
                            ptx::mbar_wait(dq_done, 0);  // the W ring's last reads are done
                            // The thread that issues the copies acquires every
                            // contributor's flag itself (then one proxy fence
                            // orders the acquired data before its async-proxy
                            // reads), each copy issued as soon as its flag is up.
                            ptx::mbar_arrive_expect_tx(fin_bar, nb * part_bytes);
                            uint32_t pending = (1u << nb) - 1u;
                            while (pending) {
                                for (uint32_t b = 0; b < nb; ++b) {
                                    const uint32_t fc = kPair ? 2 * (c0 + b) + rank : c0 + b;
                                    if (!((pending >> b) & 1u) || ptx::ld_acquire_u32(p.flags + fc) == 0) continue;
                                    p.flags[fc] = 0;
                                    ptx::fence_proxy_async();  // acquired data + prior generic SMEM reads vs TMA
                                    ptx::bulk_g2s(smem_base + b * part_bytes, p.parts + uint64_t(fc) * kSlotCellsK + kSmallCells,
                                                  part_bytes, fin_bar, ptx::policy_evict_first());
                                    pending &= ~(1u << b);
                                }
                                if (pending) __nanosleep(32);
                            }
                        }
                        if (nb) {
                            ptx::mbar_wait(fin_bar, fin_ph);
                            fin_ph ^= 1;
                        }
#ifdef LQG_TRACE_PRO
                        if (et == 0) LQG_T(11);
#endif
                        if (!last_batch) {
                            // running sum back into the accumulator for the next batch
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
                                ptx::tmem_st_x16(acc_taddr + ch * 16, sum);
                            }
                            ptx::tmem_st_wait();
                            epi_bar();  // ring reads done before the next batch
                        } else {
                            // Last batch: the team finish. This is the CTA's last
                            // segment, so the 8 dequant warps are idle: they take
                            // two of every three chunks (each warp reads its own
                            // TMEM sub-partition, warp % 4), which cuts the
                            // serial tail of the launch.
                            epi_bar();  // token scales, gathered partials seen by et 0
                            if (et == 0) {
                                team_info[0] = tile;
                                team_info[1] = acc_taddr & 0xFFFFu;
                                team_info[2] = nb;
                                ptx::tc_fence_before();
                                ptx::mbar_arrive(team_ready);  // release: team_info, ts_s, SMEM partials
                                LQG_T(8);
                            }
                            finish_chunks<kKind, kFan>(p, 0, 3, nchunks, acc_taddr, sm4, nb, part_bytes, row, n, m0,
                                                       mlim, cs, ts_s);
                            ptx::mbar_wait(team_done, 0);  // the dequant warps' chunks are read
                            ptx::tc_fence_after();
                            break;
                        }
                    }
#ifdef LQG_TRACE_PRO
                    if (et == 0) LQG_T(14);
#endif
                }
                release_acc(cur_as);
            }
            epi_bar();  // ts_s reuse
#ifdef LQG_TRACE_SEG
            if (et == 0) LQG_SEGT(eidx, 5);
            ++eidx;
#endif
        }
#ifdef LQG_TRACE_PRO
        if (et == 0) LQG_T(13);
#endif
    }

    ptx::tc_fence_before();
    __syncwarp();  // reconverge after the roles' try_wait loops (aligned barrier)
    __syncthreads();
#ifdef LQG_TRACE_PRO
    if (threadIdx.x == 0) LQG_T(12);
#endif
    ptx::tc_fence_after();
    if (kPair) ptx::cluster_sync();  // the leader's MMAs into this CTA's TMEM are complete
    if (warp == kWarpMMA) {
        if (kPair)
            ptx::tmem_dealloc_pair(tmem_base, kTmemCols);
        else
            ptx::tmem_dealloc(tmem_base, kTmemCols);
    }
}

}  // namespace lqg
