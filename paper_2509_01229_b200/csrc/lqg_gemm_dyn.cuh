// Decode-shaped W4A8 GEMM (one token tile, BN <= 32) with dynamic work
// claiming: the same warp-specialized mainloop as lqg_w4a8_gemm_kernel, but
// the (weight tile, k-range) work units are claimed dynamically from a
// counter instead of following a static stream-K split.
//
// Why: at small M the GEMM is a pure weight stream, and in a sequence of
// GEMMs under PDL the CTAs of one launch start up to several microseconds
// apart (each waits for the previous launch's CTA on its SM to exit). With a
// static schedule every CTA does the same amount of work, so the start spread
// becomes an equal finish spread and is inherited by the next launch. Here the
// grid has one persistent CTA per SM; after two statically assigned units each
// CTA claims the next unit from a counter in the workspace, so late starters
// simply process fewer units.
//
// Work unit u = (k-range ub = u / NT, weight tile nt = u % NT): k-major, so
// the units of one tile are spread over the whole launch and the tile's last
// k-range (its "finisher") is claimed after all of its contributors. A
// contributor publishes its INT32 partial into its own cells; the finisher
// sums the published partials while its own MMAs run, adds its accumulator
// and applies the reference epilogue (quant.cpp:125-127). Integer
// addition is associative, so the result is bit-identical to the reference's
// fixed-order sum in any arrival order.
//
// Reference semantics: lq::gemm_w4a8_accum / lq::gemm_w4a8
// (/root/reference/proj/src/gemm.cpp:138-223).
#pragma once
#include "lqg_gemm.cuh"

namespace lqg {

constexpr uint32_t kUidSlots = 32;          // unit-id ring (>= stages + a-slots + 2 acc + 1)
constexpr uint32_t kUidEnd = 0xFFFFFFFFu;   // "no more units"
constexpr uint32_t kDynMaxBN = 32;          // a row's partial sums live in registers
constexpr uint32_t kDynMaxUPT = 9;          // k-ranges per tile: <= 2 batches of partials per finisher
constexpr uint32_t kDynCtlBytes = 4096;     // barriers + misc after the ring

#ifdef LQG_TRACE
__device__ __forceinline__ uint64_t dyn_now() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t dyn_smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#define DYN_SLOT(e) g_lqg_trace[(p.trace_slot * 160 + dyn_smid()) * 16 + (e)]
#define DYN_T(e) do { if ((threadIdx.x & 31) == 0) DYN_SLOT(e) = dyn_now(); } while (0)
#define DYN_ADD(e, v) do { if ((threadIdx.x & 31) == 0) DYN_SLOT(e) += (v); } while (0)
#define DYN_NOW() dyn_now()
#else
#define DYN_T(e) ((void)0)
#define DYN_ADD(e, v) ((void)0)
#define DYN_NOW() 0ull
#endif

// k-major unit order: u = ub * NT + nt. Unit u of tile nt covers k-range
// r = (ub + nt) % UPT, i.e. k-blocks [r * unit_kb, +nkb), walked from a
// per-tile rotation: the ~#SM units in flight at any time then read
// different activation k-blocks (no L2 hot spot on one X slice). The
// reduction order is irrelevant (exact integer sums).
__device__ __forceinline__ void unit_coords(uint32_t u, const GemmParams& p, uint32_t& nt,
                                            uint32_t& ub, uint32_t& kb0, uint32_t& nkb) {
    ub = u / p.NT;
    nt = u - ub * p.NT;
    uint32_t r = ub + nt % p.units_per_tile;
    if (r >= p.units_per_tile) r -= p.units_per_tile;
    kb0 = r * p.unit_kb;
    nkb = min(p.unit_kb, p.KB - kb0);
}

// The k-blocks of one unit in issue order (producer side only: dequant and
// MMA consume ring slots in order, whatever k-block they hold).
struct UnitWalk {
    uint32_t nt, kb0, nkb, j, rot;
    __device__ __forceinline__ void set(uint32_t u, const GemmParams& p) {
        uint32_t ub;
        unit_coords(u, p, nt, ub, kb0, nkb);
        j = 0;
        rot = (nt * 7u) % nkb;
    }
    __device__ __forceinline__ uint32_t kb() const {
        const uint32_t t = j + rot;
        return kb0 + (t >= nkb ? t - nkb : t);
    }
    __device__ __forceinline__ bool step() { return ++j == nkb; }  // true at the unit's end
};

__device__ __forceinline__ bool cell_pending(const int4& x) {
    return x.x == INT32_MIN || x.y == INT32_MIN || x.z == INT32_MIN || x.w == INT32_MIN;
}

__global__ void __launch_bounds__(kThreads, 1)
    lqg_w4a8_dyn_kernel(const __grid_constant__ CUtensorMap tmap_x, const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t pad = (1024 - (raw_addr & 1023)) & 1023;
    uint8_t* smem = smem_raw + pad;
    const uint32_t smem_base = raw_addr + pad;

    const uint32_t S = p.stages;
    const uint32_t ring_bytes = S * p.stage_bytes;
    const uint32_t bar_base = smem_base + ring_bytes;
    auto wfull_bar = [&](uint32_t s) { return bar_base + 8 * s; };
    auto xfull_bar = [&](uint32_t s) { return bar_base + 8 * (kMaxStages + s); };
    auto empty_bar = [&](uint32_t s) { return bar_base + 8 * (2 * kMaxStages + s); };
    constexpr uint32_t kB = 3 * kMaxStages;
    auto afull_bar = [&](uint32_t a) { return bar_base + 8 * (kB + a); };
    auto aempty_bar = [&](uint32_t a) { return bar_base + 8 * (kB + kMaxASlots + a); };
    auto accfull_bar = [&](uint32_t a) { return bar_base + 8 * (kB + 2 * kMaxASlots + a); };
    auto accempty_bar = [&](uint32_t a) { return bar_base + 8 * (kB + 2 * kMaxASlots + 2 + a); };
    constexpr uint32_t kU = kB + 2 * kMaxASlots + 4;
    auto uidfull_bar = [&](uint32_t i) { return bar_base + 8 * (kU + i); };
    auto uidempty_bar = [&](uint32_t i) { return bar_base + 8 * (kU + kUidSlots + i); };
    constexpr uint32_t kMisc = (8 * (kU + 2 * kUidSlots) + 63) / 64 * 64;
    uint8_t* misc = smem + ring_bytes + kMisc;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(misc);
    volatile uint32_t* uid_s = reinterpret_cast<volatile uint32_t*>(misc + 64);
    float* ts_s = reinterpret_cast<float*>(misc + 64 + 4 * kUidSlots);

    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t KB = p.KB;
    const TmemPlan tp = tmem_plan(p.BN, 512);
    const uint32_t x_bytes = p.BN * kKBlock;

    if (threadIdx.x == 0) {
        DYN_T(0);
#ifdef LQG_TRACE
        for (uint32_t e = 8; e < 16; ++e) DYN_SLOT(e) = 0;
#endif
        for (uint32_t s = 0; s < S; ++s) {
            ptx::mbar_init(wfull_bar(s), 1);
            ptx::mbar_init(xfull_bar(s), 1);
            ptx::mbar_init(empty_bar(s), 1);
        }
        for (uint32_t a = 0; a < kMaxASlots; ++a) {
            ptx::mbar_init(afull_bar(a), 8);
            ptx::mbar_init(aempty_bar(a), 1);
        }
        for (uint32_t a = 0; a < 2; ++a) {
            ptx::mbar_init(accfull_bar(a), 1);
            ptx::mbar_init(accempty_bar(a), 4);
        }
        // consumers of every unit id: MMA lane, 8 dequant warps, 4 epilogue warps
        for (uint32_t i = 0; i < kUidSlots; ++i) {
            ptx::mbar_init(uidfull_bar(i), 1);
            ptx::mbar_init(uidempty_bar(i), 13);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    if (threadIdx.x == 0) ptx::launch_dependents();
    if (threadIdx.x == 0) DYN_T(1);

    if (warp == 0) {
        // ------------------------------------------------ scheduler + TMA producer
        // Warp-uniform loop: every lane waits on the barriers, lane 0 issues.
        {
            if (lane == 0) ptx::prefetch_tmap(&tmap_x);
            const uint64_t pol_w = ptx::policy_evict_first();
            const uint64_t pol_x = ptx::policy_evict_last();
            const uint32_t atom_bytes = p.BN * kXAtom;
            const uint32_t G = gridDim.x;
            const uint32_t S0 = p.static_units;                     // units [0, S0): CTA c gets c, c+G, ...
            const uint32_t n_units = p.NT * p.units_per_tile;
            const uint32_t last_ticket = (n_units - S0) + G - 1;   // every CTA fails exactly one claim
            uint32_t static_next = blockIdx.x;
            bool claim_live = false;  // a claim is in flight (issued one unit ahead)
            uint32_t ticket = 0;
            uint32_t us = 0, uph = 0;
            auto push_uid = [&](uint32_t v) {
                const uint64_t t0 = DYN_NOW();
                ptx::mbar_wait(uidempty_bar(us), uph ^ 1);
                DYN_ADD(10, DYN_NOW() - t0);
                if (lane == 0) {
                    uid_s[us] = v;
                    ptx::mbar_arrive(uidfull_bar(us));
                }
                __syncwarp();
                if (++us == kUidSlots) {
                    us = 0;
                    uph ^= 1;
                }
            };
            // Next unit of this CTA. Static units first; then tickets from the
            // per-workspace counter (monotonic claims; only after the PDL wait,
            // when the previous launch has reset the counter). The holder of the
            // last ticket resets it for the next launch.
            auto next_unit = [&]() -> uint32_t {
                if (static_next < S0) {
                    const uint32_t u = static_next;
                    static_next += G;
                    if (static_next >= S0) {
                        if (lane == 0) ticket = atomicAdd(p.dcnt, 1u);  // claim ahead
                        claim_live = true;
                    }
                    return u;
                }
                if (!claim_live) {
                    if (lane == 0) ticket = atomicAdd(p.dcnt, 1u);
                    claim_live = true;
                }
#ifdef LQG_TRACE
                const uint64_t t0 = DYN_NOW();
                uint32_t t;
                asm volatile("mov.u32 %0, %1;" : "=r"(t) : "r"(ticket));  // waits for the atomic's return
                t = __shfl_sync(0xffffffffu, t, 0);
                DYN_ADD(8, DYN_NOW() - t0);
#else
                const uint32_t t = __shfl_sync(0xffffffffu, ticket, 0);  // waits for the atomic's return
#endif
                claim_live = false;
                if (lane == 0 && t == last_ticket) atomicExch(p.dcnt, 0u);
                if (S0 + t < n_units) {
                    if (lane == 0) ticket = atomicAdd(p.dcnt, 1u);  // claim ahead
                    claim_live = true;
                    return S0 + t;
                }
                return kUidEnd;
            };
            UnitWalk ww;
            auto w_set = [&](uint32_t u) { ww.set(u, p); };
            auto w_issue = [&](uint32_t st) {
                if (lane == 0) {
                    ptx::mbar_arrive_expect_tx(wfull_bar(st), p.chunk_bytes);
                    ptx::bulk_g2s(smem_base + st * p.stage_bytes + x_bytes,
                                  p.wimg + (uint64_t(ww.nt) * KB + ww.kb()) * p.chunk_bytes, p.chunk_bytes,
                                  wfull_bar(st), pol_w);
                }
            };
            auto x_issue = [&](uint32_t st, uint32_t kb) {
                if (lane != 0) return;
                const uint32_t slot = smem_base + st * p.stage_bytes;
                ptx::mbar_arrive_expect_tx(xfull_bar(st), x_bytes);
                const int32_t k0 = int32_t(kb * kKBlock);
                ptx::tma_2d_g2s(slot, &tmap_x, k0, 0, xfull_bar(st), pol_x);
                ptx::tma_2d_g2s(slot + atom_bytes, &tmap_x, k0 + int32_t(kXAtom), 0, xfull_bar(st),
                                pol_x);
            };
            // Weights are static: the chunks of this CTA's static units fill the
            // ring before the PDL wait (overlapping the previous kernel's tail).
            const uint32_t u0 = blockIdx.x;
            static_next += G;
            push_uid(u0);
            w_set(u0);
            uint32_t issued = 0;
            bool need_next = false;
            while (issued < S) {
                if (need_next) {
                    if (static_next >= S0) break;  // further units need a claim
                    const uint32_t u = static_next;
                    static_next += G;
                    push_uid(u);
                    w_set(u);
                    need_next = false;
                }
                w_issue(issued++);
                if (ww.step()) need_next = true;
            }
            ptx::griddep_wait();
            DYN_T(2);
            {
                // activations of the chunks issued so far (static units, in order)
                uint32_t xu = u0;
                UnitWalk xw;
                xw.set(xu, p);
                for (uint32_t i = 0; i < issued; ++i) {
                    x_issue(i, xw.kb());
                    if (xw.step() && i + 1 < issued) {
                        xu += G;
                        xw.set(xu, p);
                    }
                }
            }
            if (static_next >= S0 && !claim_live) {
                if (lane == 0) ticket = atomicAdd(p.dcnt, 1u);
                claim_live = true;
            }
            uint32_t s = issued == S ? 0 : issued, ph = issued == S ? 1 : 0;
            for (;;) {
                if (need_next) {
                    const uint32_t u = next_unit();
                    push_uid(u);
                    if (u == kUidEnd) break;
                    w_set(u);
                    need_next = false;
                }
                const uint64_t t0 = DYN_NOW();
                ptx::mbar_wait(empty_bar(s), ph ^ 1);
                DYN_ADD(12, DYN_NOW() - t0);
                w_issue(s);
                x_issue(s, ww.kb());
                if (ww.step()) need_next = true;
                if (++s == S) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        {
            const uint32_t idesc = ptx::idesc_i8(kTileN, p.BN);
            const uint64_t desc0 = ptx::sw128_kmajor_desc(smem_base);
            const uint32_t stage_desc = p.stage_bytes >> 4;
            const uint32_t atom_desc = (p.BN * kXAtom) >> 4;
            uint32_t us = 0, uph = 0, s = 0, ph = 0, a = 0, aph = 0, as = 0, acc_ph = 0;
            for (;;) {
                ptx::mbar_wait(uidfull_bar(us), uph);
                const uint32_t u = uid_s[us];
                if (u == kUidEnd) break;
                uint32_t nt, ub, kb0, nkb;
                unit_coords(u, p, nt, ub, kb0, nkb);
                const uint64_t t0 = DYN_NOW();
                ptx::mbar_wait(accempty_bar(as), acc_ph ^ 1);
                DYN_ADD(11, DYN_NOW() - t0);
                DYN_ADD(9, 1);
                const uint32_t d_tmem = tmem_base + as * tp.acc_stride;
                for (uint32_t j = 0; j < nkb; ++j) {
                    const uint64_t ta = DYN_NOW();
                    ptx::mbar_wait(afull_bar(a), aph);
                    const uint64_t tb = DYN_NOW();
                    ptx::mbar_wait(xfull_bar(s), ph);
                    DYN_ADD(13, tb - ta);
                    DYN_ADD(14, DYN_NOW() - tb);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t a_tmem = tmem_base + tp.a_base + a * kACols;
                        const uint64_t bdesc = desc0 + uint64_t(s * stage_desc);
#pragma unroll
                        for (uint32_t k8 = 0; k8 < kSubBlocks; ++k8)
                            ptx::mma_i8_ts(d_tmem, a_tmem + k8 * 8,
                                           bdesc + (k8 / 4) * atom_desc + (k8 % 4) * 2, idesc,
                                           (j == 0 && k8 == 0) ? 0u : 1u);
                        ptx::mma_commit(empty_bar(s));
                        ptx::mma_commit(aempty_bar(a));
                        if (j + 1 == nkb) ptx::mma_commit(accfull_bar(as));
                    }
                    __syncwarp();
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                    if (++a == tp.a_slots) {
                        a = 0;
                        aph ^= 1;
                    }
                }
                if (lane == 0) ptx::mbar_arrive(uidempty_bar(us));
                if (++us == kUidSlots) {
                    us = 0;
                    uph ^= 1;
                }
                if (++as == tp.acc_stages) {
                    as = 0;
                    acc_ph ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp >= kDequantWarp0 && warp < kEpiWarp0) {
        // ------------------------------------------------------------ dequant WGs
        const uint32_t wg = (warp - kDequantWarp0) / 4;
        const uint32_t sp = warp % 4;
        const uint32_t row = sp * 32 + lane;
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t p_shift = param_shift(p.P);
        constexpr uint32_t kHalf = kSubBlocks / 2;
        const uint8_t* ring_w = smem + x_bytes;
        const uint32_t a_base = tmem_base + lane_addr + tp.a_base + wg * kHalf * 8;
        uint32_t us = 0, uph = 0, s = 0, ph = 0, a = 0, aph = 0;
        for (;;) {
            ptx::mbar_wait(uidfull_bar(us), uph);
            const uint32_t u = uid_s[us];
            if (u == kUidEnd) break;
            uint32_t nt, ub, kb0, nkb;
            unit_coords(u, p, nt, ub, kb0, nkb);
            for (uint32_t j = 0; j < nkb; ++j) {
                ptx::mbar_wait(wfull_bar(s), ph);
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
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(uidempty_bar(us));
            if (++us == kUidSlots) {
                us = 0;
                uph ^= 1;
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ------------------------------------------------------------ epilogue
        // Split tiles: every contributor unit (k-range ub < UPT-1 of its tile)
        // publishes its INT32 partial into its own cells in `parts` ([chunk]
        // [row][16], INT32_MIN = not published; |partial| < 2^31 - 1 so it
        // never occurs as a value) and moves on: no fence, no counter, no wait.
        // The finisher (the tile's last k-range, claimed after every
        // contributor because claims are monotonic) sums the published
        // partials in batches while its own MMAs run, then adds its
        // accumulator and any late partial (spinning only on lower-numbered
        // units: no deadlock), applies the epilogue and restores the
        // sentinels. Each thread owns one weight row end to end.
        const uint32_t sp = warp % 4;
        const uint32_t row = sp * 32 + lane;
        const uint32_t lane_addr = (sp * 32) << 16;
        const uint32_t et = threadIdx.x - kEpiWarp0 * 32;  // 0..127
        const uint32_t nchunks = p.BN / 16;                 // 1 or 2
        const bool scaled = p.out_kind != kOutAcc;
        const uint32_t UPT = p.units_per_tile, NT = p.NT;
        const bool split = UPT > 1;
        const uint64_t slot_cells = uint64_t(p.BN) * kTileN;
        auto data_cell = [&](uint32_t slot, uint32_t ch) {
            return reinterpret_cast<int4*>(p.parts + uint64_t(slot) * slot_cells + (ch * kTileN + row) * 16);
        };
        const int4 kSent4 = make_int4(INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN);
        ptx::griddep_wait();
        if (scaled)
            for (uint32_t j = et; j < p.BN; j += 128) ts_s[j] = j < p.M ? p.ts[j] : 0.f;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        uint32_t us = 0, uph = 0, as = 0, acc_ph = 0;
        for (;;) {
            ptx::mbar_wait(uidfull_bar(us), uph);
            const uint32_t u = uid_s[us];
            if (u == kUidEnd) break;
            uint32_t nt, ub, kb0, nkb;
            unit_coords(u, p, nt, ub, kb0, nkb);
            const uint32_t n = nt * kTileN + row;
            const double cs = scaled ? double(p.cs[n]) : 0.0;
            const bool finisher = split && ub + 1 == UPT;
            int32_t pre[2][16];
            uint32_t pend[2] = {0u, 0u};
#pragma unroll
            for (uint32_t ch = 0; ch < 2; ++ch)
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) pre[ch][j] = 0;
            if (finisher) {
#pragma unroll
                for (uint32_t ch = 0; ch < 2; ++ch) {
                    if (ch >= nchunks) break;
                    for (uint32_t c0 = 0; c0 + 1 < UPT; c0 += 4) {
                        const uint32_t nb = min(4u, UPT - 1 - c0);
                        int4 cv[4][4];
#pragma unroll
                        for (uint32_t b = 0; b < 4; ++b)
#pragma unroll
                            for (uint32_t q = 0; q < 4; ++q)
                                cv[b][q] = b < nb ? __ldcg(data_cell((c0 + b) * NT + nt, ch) + q) : kSent4;
#pragma unroll
                        for (uint32_t b = 0; b < 4; ++b) {
                            bool ready = b < nb;
#pragma unroll
                            for (uint32_t q = 0; q < 4; ++q) ready = ready && !cell_pending(cv[b][q]);
                            if (ready) {
#pragma unroll
                                for (uint32_t q = 0; q < 4; ++q) {
                                    pre[ch][4 * q] += cv[b][q].x;
                                    pre[ch][4 * q + 1] += cv[b][q].y;
                                    pre[ch][4 * q + 2] += cv[b][q].z;
                                    pre[ch][4 * q + 3] += cv[b][q].w;
                                    __stcg(data_cell((c0 + b) * NT + nt, ch) + q, kSent4);
                                }
                            } else if (b < nb) {
                                pend[ch] |= 1u << (c0 + b);
                            }
                        }
                    }
                }
            }
            ptx::mbar_wait(accfull_bar(as), acc_ph);
            ptx::tc_fence_after();
            const uint32_t acc_taddr = tmem_base + lane_addr + as * tp.acc_stride;
            const uint32_t cur_as = as;
            if (++as == tp.acc_stages) {
                as = 0;
                acc_ph ^= 1;
            }
            uint32_t v[2][16];
            ptx::tmem_ld_x16(acc_taddr, v[0]);
            if (nchunks > 1) ptx::tmem_ld_x16(acc_taddr + 16, v[1]);
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(accempty_bar(cur_as));
#pragma unroll
            for (uint32_t ch = 0; ch < 2; ++ch) {
                if (ch >= nchunks) break;
                if (split && !finisher) {
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q)
                        __stcg(data_cell(u, ch) + q, make_int4(int32_t(v[ch][4 * q]), int32_t(v[ch][4 * q + 1]),
                                                               int32_t(v[ch][4 * q + 2]), int32_t(v[ch][4 * q + 3])));
                    continue;
                }
                int32_t sum[16];
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) sum[j] = int32_t(v[ch][j]) + pre[ch][j];
                uint32_t mask = pend[ch];
                while (mask) {
                    const uint32_t c = __ffs(mask) - 1;
                    int4* cell = data_cell(c * NT + nt, ch);
                    int4 cv[4];
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) cv[q] = ptx::ld_relaxed_v4(cell + q);
                    bool ready = true;
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) ready = ready && !cell_pending(cv[q]);
                    if (!ready) {
                        __nanosleep(32);
                        continue;
                    }
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) {
                        sum[4 * q] += cv[q].x;
                        sum[4 * q + 1] += cv[q].y;
                        sum[4 * q + 2] += cv[q].z;
                        sum[4 * q + 3] += cv[q].w;
                        __stcg(cell + q, kSent4);
                    }
                    mask &= mask - 1;
                }
                if (n < p.N) store_chunk(p, ch * 16, n, sum, cs, ts_s + ch * 16);
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(uidempty_bar(us));
            if (++us == kUidSlots) {
                us = 0;
                uph ^= 1;
            }
        }
    }

    if (threadIdx.x == kEpiWarp0 * 32) DYN_T(5);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) DYN_T(6);
    if (warp == 1) ptx::tmem_dealloc(tmem_base, 512);
}

}  // namespace lqg
