// C-ABI implementation of include/lqg.h: validation with the reference's
// semantics, host prepack into the device image, launch configuration and
// the host-buffer staging path. See lqg_gemm.cuh for the kernel design.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/lqg.h"
#include "lqg_aux.cuh"
#include "lqg_launch.h"
#include "lqg_layout.h"

using namespace lqg;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

struct Status {
    int code;
};

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define LQG_CUDA(expr)                                                                       \
    do {                                                                                     \
        cudaError_t e__ = (expr);                                                            \
        if (e__ != cudaSuccess)                                                              \
            return set_err(LQG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int check_device(int dev, int* num_sms) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return set_err(LQG_EUNSUPPORTED, "no CUDA device available (liblqg has no CPU fallback)");
    if (dev < 0 || dev >= count) return set_err(LQG_EVALIDATION, "device index out of range");
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return set_err(LQG_EUNSUPPORTED, "liblqg is built for sm_100a (B200); device has sm_" +
                                             std::to_string(major) + std::to_string(minor));
    if (num_sms) cudaDeviceGetAttribute(num_sms, cudaDevAttrMultiProcessorCount, dev);
    return LQG_OK;
}

// ---------------------------------------------------------------- tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// ---------------------------------------------------------------- workspace
constexpr uint32_t kMaxSlots = 160;  // >= SM count of any sm_100 part
constexpr uint64_t kSlotCells = kSlotCellsK;  // INT32 partial-sum cells per CTA (lqg_gemm.cuh)

}  // namespace

struct lqg_workspace {
    int device = 0;
    int32_t* parts = nullptr;  // [kMaxSlots][kSlotCells] split-K partials (INT32_MIN =
                               // not published), then kMaxSlots "published" flags (0)
};

struct lqg_weights {
    int device = 0;
    int num_sms = 148;
    ImageGeom geom{};
    uint8_t* d_img = nullptr;
    uint64_t img_bytes = 0;
    float* d_cs = nullptr;
};

namespace {

// Runs `f` with this thread's stream-capture mode relaxed, so that the
// one-off allocations and initialisation below are legal while another
// stream (e.g. a CUDA-graph capture of the first GEMMs) is capturing.
template <typename F>
auto relaxed_capture(F&& f) {
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    auto r = f();
    cudaThreadExchangeStreamCaptureMode(&mode);
    return r;
}

int workspace_create(int dev, lqg_workspace** out) {
    return relaxed_capture([&]() -> int {
        auto* w = new lqg_workspace();
        w->device = dev;
        DeviceGuard g(dev);
        cudaStream_t st = nullptr;
        if (cudaMalloc(&w->parts, (kMaxSlots * kSlotCells + kMaxSlots) * 4) != cudaSuccess ||
            cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
            cudaFree(w->parts);
            delete w;
            return set_err(LQG_ECUDA, "workspace allocation failed");
        }
        fill_i32_kernel<<<592, 256, 0, st>>>(w->parts, kMaxSlots * kSlotCells, INT32_MIN);
        fill_i32_kernel<<<1, 256, 0, st>>>(w->parts + kMaxSlots * kSlotCells, kMaxSlots, 0);
        const cudaError_t e = cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        if (e != cudaSuccess) {
            cudaFree(w->parts);
            delete w;
            return set_err(LQG_ECUDA, "workspace initialisation failed");
        }
        *out = w;
        return LQG_OK;
    });
}

// The default split-K workspace of a (device, stream): shared by every
// handle, created on first use and kept for the life of the process. Launches
// on one stream are ordered, so they can share one workspace; launches on
// different streams get different ones, which keeps concurrent launches
// through one (immutable) handle safe without an explicit workspace.
int default_workspace(int dev, cudaStream_t st, lqg_workspace** out) {
    struct Entry {
        int dev;
        cudaStream_t st;
        lqg_workspace* ws;
    };
    static std::mutex mu;
    static std::vector<Entry>* pool = new std::vector<Entry>();  // process lifetime
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry& e : *pool)
        if (e.dev == dev && e.st == st) {
            *out = e.ws;
            return LQG_OK;
        }
    lqg_workspace* w = nullptr;
    int rc = workspace_create(dev, &w);
    if (rc) return rc;
    pool->push_back({dev, st, w});
    *out = w;
    return LQG_OK;
}

// Reference validation, bundle.cpp:89-135 (+ FragmentDescriptor::validate,
// layout.cpp:10-22).
int validate_bundle(const lqg_bundle_view& b) {
    if (b.n < 1 || b.k < 1) return set_err(LQG_EVALIDATION, "bundle dimensions must be >= 1");
    if (b.group_size < 1) return set_err(LQG_EVALIDATION, "group_size must be >= 1");
    if (b.k % b.group_size != 0)
        return set_err(LQG_EVALIDATION, "k = " + std::to_string(b.k) +
                                            " not divisible by group_size = " +
                                            std::to_string(b.group_size));
    if (b.layout > 1) return set_err(LQG_EVALIDATION, "unknown layout flag " + std::to_string(b.layout));
    if (b.layout == LQG_LAYOUT_DUAL_MMA) {
        const auto& d = b.fragment;
        const uint32_t slab = uint32_t(d.mma_m) * d.mma_k;
        const uint32_t per_group =
            uint32_t(d.warps_per_group) * d.threads_per_warp * d.elements_per_thread_per_mma;
        if (slab != per_group)
            return set_err(LQG_EVALIDATION, "fragment descriptor mismatch: mma_m*mma_k = " +
                                                std::to_string(slab) + " but group covers " +
                                                std::to_string(per_group) + " elements");
        if (d.dual_k_span != 2 * d.mma_k)
            return set_err(LQG_EVALIDATION, "dual_k_span must be 2*mma_k");
        if (!d.warps_per_group || !d.threads_per_warp || !d.mma_m || !d.mma_k)
            return set_err(LQG_EVALIDATION, "fragment descriptor has a zero field");
        if (b.n % d.mma_m != 0)
            return set_err(LQG_EVALIDATION,
                           "dual-MMA layout needs n divisible by " + std::to_string(d.mma_m));
        if (b.k % d.dual_k_span != 0)
            return set_err(LQG_EVALIDATION,
                           "dual-MMA layout needs k divisible by " + std::to_string(d.dual_k_span));
        if (b.group_size % d.dual_k_span != 0)
            return set_err(LQG_EVALIDATION, "dual-MMA layout needs group_size divisible by " +
                                                std::to_string(d.dual_k_span) +
                                                " so each record word pair stays within one group");
    }
    const uint64_t nk = uint64_t(b.n) * b.k;
    if (!b.packed_weights || b.packed_bytes != (nk + 1) / 2)
        return set_err(LQG_EVALIDATION, "packed weight payload has wrong size");
    const uint32_t gpr = b.k / b.group_size;
    const uint64_t ng = uint64_t(b.n) * gpr;
    if (!b.group_scales || !b.group_offsets || b.n_groups != ng)
        return set_err(LQG_EVALIDATION, "group parameter arrays have wrong size");
    if (!b.channel_scales) return set_err(LQG_EVALIDATION, "channel scale array has wrong size");
    for (uint64_t i = 0; i < ng; ++i) {
        const uint32_t row = uint32_t(i / gpr), g = uint32_t(i % gpr);
        if (b.group_scales[i] < 1 || b.group_scales[i] > 16)
            return set_err(LQG_EVALIDATION, "group scale " + std::to_string(int(b.group_scales[i])) +
                                                " out of [1,16] at row " + std::to_string(row) +
                                                " group " + std::to_string(g));
        if (b.group_offsets[i] < 9 || b.group_offsets[i] > 247)
            return set_err(LQG_EVALIDATION, "group offset " +
                                                std::to_string(int(b.group_offsets[i])) +
                                                " out of [9,247] at row " + std::to_string(row) +
                                                " group " + std::to_string(g));
    }
    for (uint32_t r = 0; r < b.n; ++r) {
        const float s = b.channel_scales[r];
        if (!(s > 0.0f) || !std::isfinite(s))
            return set_err(LQG_EVALIDATION, "channel scale at row " + std::to_string(r) +
                                                " must be positive and finite");
    }
    return LQG_OK;
}

int device_layout_supported(uint32_t g) {
    if (g % 32 != 0)
        return set_err(LQG_EVALIDATION, "the sm_100a device layout needs group_size % 32 == 0 (got " +
                                            std::to_string(g) + ")");
    return LQG_OK;
}

// Logical code (row, col) of a bundle in either layout (bundle.cpp:59-87).
struct CodeReader {
    const lqg_bundle_view& b;
    uint8_t at(uint32_t row, uint32_t col) const {
        if (b.layout == LQG_LAYOUT_PLAIN) {
            const uint64_t idx = uint64_t(row) * b.k + col;
            const uint8_t byte = b.packed_weights[idx / 2];
            return (idx % 2 == 0) ? (byte & 0x0F) : (byte >> 4);
        }
        const auto& d = b.fragment;
        const uint32_t band = row / d.mma_m, r_in = row % d.mma_m;
        const uint32_t warp = r_in / 16, r = (r_in % 16) / 8, row_quarter = r_in % 8;
        const uint32_t pair = col / d.dual_k_span, col_in = col % d.dual_k_span;
        const uint32_t half = col_in / d.mma_k, c32 = col_in % d.mma_k;
        const uint32_t bsel = c32 / 16;
        const uint32_t thread = 4 * row_quarter + (c32 % 16) / 4;
        const uint32_t j = c32 % 4;
        const uint64_t band_bytes = uint64_t(d.mma_m) * b.k / 2;
        const uint64_t record = (uint64_t(pair) * d.warps_per_group + warp) * d.threads_per_warp + thread;
        const uint64_t byte_idx = band * band_bytes + record * 16 + (2 * half + r) * 4 + j;
        const uint8_t byte = b.packed_weights[byte_idx];
        return bsel == 0 ? (byte & 0x0F) : (byte >> 4);
    }
};

// Host prepack: bundle (either layout) -> device image (lqg_layout.h).
void prepack_host(const lqg_bundle_view& b, const ImageGeom& G, std::vector<uint8_t>& img) {
    img.assign(uint64_t(G.NT) * G.KB * G.chunk_bytes, 0);
    // padding params (s=1, a=128)
    for (uint64_t ch = 0; ch < uint64_t(G.NT) * G.KB; ++ch)
        for (uint32_t i = 0; i < 128 * G.P; ++i) {
            uint8_t* p = img.data() + ch * G.chunk_bytes + kCodeBytes + 2 * i;
            p[0] = 1;
            p[1] = 128;
        }
    CodeReader rd{b};
    const uint32_t gpr = b.k / b.group_size;
    std::vector<uint8_t> rowcodes(b.k);
    for (uint32_t row = 0; row < b.n; ++row) {
        if (b.layout == LQG_LAYOUT_PLAIN && (uint64_t(row) * b.k) % 2 == 0) {
            const uint8_t* src = b.packed_weights + uint64_t(row) * b.k / 2;
            for (uint32_t c = 0; c + 1 < b.k; c += 2) {
                rowcodes[c] = src[c / 2] & 0x0F;
                rowcodes[c + 1] = src[c / 2] >> 4;
            }
            if (b.k % 2) rowcodes[b.k - 1] = src[(b.k - 1) / 2] & 0x0F;
        } else {
            for (uint32_t c = 0; c < b.k; ++c) rowcodes[c] = rd.at(row, c);
        }
        for (uint32_t k0 = 0; k0 < b.k; k0 += 8) {
            uint32_t word = 0;
            for (uint32_t j = 0; j < 4; ++j) {
                const uint32_t lo = k0 + j < b.k ? rowcodes[k0 + j] : 0;
                const uint32_t hi = k0 + j + 4 < b.k ? rowcodes[k0 + j + 4] : 0;
                word |= (lo | (hi << 4)) << (8 * j);
            }
            const uint32_t kb = k0 / kKBlock, c = (k0 % kKBlock) / 32, wsub = (k0 % 32) / 8;
            std::memcpy(img.data() + code_offset(G.chunk_bytes, G.KB, row, kb, c) + wsub * 4, &word, 4);
        }
        const uint32_t sub_per_p = kSubBlocks / G.P;
        for (uint32_t k0 = 0; k0 < b.k; k0 += 32) {
            const uint32_t kb = k0 / kKBlock, c = (k0 % kKBlock) / 32;
            if (c % sub_per_p) continue;
            const uint32_t gi = k0 / b.group_size;
            uint8_t* p = img.data() + param_offset(G.chunk_bytes, G.KB, row, kb, c / sub_per_p);
            p[0] = b.group_scales[uint64_t(row) * gpr + gi];
            p[1] = b.group_offsets[uint64_t(row) * gpr + gi];
        }
    }
}

int alloc_weights(int dev, const ImageGeom& G, lqg_weights** out) {
    auto* w = new lqg_weights();
    w->device = dev;
    w->geom = G;
    w->img_bytes = uint64_t(G.NT) * G.KB * G.chunk_bytes;
    int rc = check_device(dev, &w->num_sms);
    if (rc) {
        delete w;
        return rc;
    }
    DeviceGuard g(dev);
    if (cudaMalloc(&w->d_img, w->img_bytes) != cudaSuccess ||
        cudaMalloc(&w->d_cs, uint64_t(G.NT) * kTileN * 4) != cudaSuccess) {
        cudaFree(w->d_img);
        delete w;
        return set_err(LQG_ECUDA, "weight image allocation failed");
    }
    *out = w;
    return LQG_OK;
}

// Token tile: <= 192 so that the INT32 accumulator stays double-buffered in
// TMEM (2 x 192 columns + a 2-slot A ring, see tmem_plan).
constexpr uint32_t kMaxTileM = 192;
// CTA pairs from this many tokens (largest group), also with a single token
// tile: one M = 256 MMA per k-block serves two SMs, which halves the MMA
// warp's per-k-block overhead per SM (LLaMA-2-70B 4-GEMM step on B200:
// M = 128 117 -> 110 us, M = 256 176 -> 159 us; M = 16 unchanged either way).
// Below 80 tokens one-CTA tiles are faster (tools/sched_sweep.py, 4-GEMM
// steps: 70B at M = 48 89.1 -> 84.3 us, M = 64 89.7 -> 88.6; 7B at M = 48
// 53.2 -> 47.1 and M = 64 53.2 -> 49.3 with pick_tiles' rule D), from 96
// tokens pairs win (70B M = 96 94.8 vs 97.8 us without).
constexpr uint32_t kPairMinM = 80;
constexpr uint32_t kDecodeWStages = 6;  // W ring depth for token tiles <= 32
// Dynamic shared memory: the two rings, then barriers / schedule / token scales.

// 1024-byte alignment pad + mbarriers + misc (holder, token scales, output staging)
constexpr uint32_t kSmemMisc = (1024 + 8 * kNumBarriers + 8 + kMiscBytes + 1023) / 1024 * 1024;

// Launch-schedule knobs: token-tile cap, CTA-pair policy, ring split, grid.
// Results never depend on them (every setting is bit-exact, tested); they
// only move the schedule. Defaults are the measured best on B200; tools and
// tests change them through lqg_tune_set (process-wide, no environment reads).
enum TuneId : int {
    kTuneMaxBN, kTunePairMinM, kTunePair, kTunePairSingleTile, kTuneXRingBytes, kTuneMaxXStages,
    kTuneMaxWStages, kTuneGrid, kTuneRasterGM, kTuneNoDP, kTuneNoPDL, kTuneAccStages, kTuneHostChunkM, kTuneHostChunks, kTuneNoQuad, kTuneAutoTile, kTuneCount
};
struct TuneDef {
    const char* name;
    int64_t dflt, lo, hi;
};
constexpr TuneDef kTuneDefs[kTuneCount] = {
    {"max_bn", kMaxTileM, 16, kMaxTileM},          // token-tile cap
    {"pair_min_m", kPairMinM, 1, 1 << 30},         // CTA pairs from this many tokens
    {"pair", -1, -1, 1},                           // -1 auto, 0 never, 1 wherever legal
    {"pair_single_tile", 1, 0, 1},                 // allow pairs with one token tile
    {"x_ring_bytes", 0, 0, kSmemMax},              // 0 = balanced rings; else reserve for X
    {"max_x_stages", kMaxStages, 2, kMaxStages},
    {"max_w_stages", kMaxStages, 2, kMaxStages},
    {"grid", 0, 0, kMaxSlots},                     // 0 = one CTA per SM
    {"raster_gm", 0, 0, 1 << 20},                  // 0 = derived
    {"no_dp", 0, 0, 1},                            // stream-K over all tiles
    {"no_pdl", 0, 0, 1},                           // no programmatic dependent launch
    {"acc_stages", 2, 1, 2},                       // accumulator stages in TMEM (the rest is A ring)
    {"host_chunk_m", 384, 1, 1 << 30},             // host-buffer calls of >= this many rows are pipelined
    {"host_chunks", 6, 1, 8},                      // ... in this many row chunks
    {"no_quad", 0, 0, 1},                          // 1: split tiles exchange through L2 even where a 4-CTA cluster fits
    {"auto_tile", 1, 0, 1},                        // token-tile / pair rules for few or short-K tiles (see pick_tiles)
};
std::atomic<int64_t> g_tune[kTuneCount] = {
    {kTuneDefs[0].dflt}, {kTuneDefs[1].dflt}, {kTuneDefs[2].dflt}, {kTuneDefs[3].dflt},
    {kTuneDefs[4].dflt}, {kTuneDefs[5].dflt}, {kTuneDefs[6].dflt}, {kTuneDefs[7].dflt},
    {kTuneDefs[8].dflt}, {kTuneDefs[9].dflt}, {kTuneDefs[10].dflt}, {kTuneDefs[11].dflt},
    {kTuneDefs[12].dflt}, {kTuneDefs[13].dflt}, {kTuneDefs[14].dflt}, {kTuneDefs[15].dflt}};

struct Knobs {
    uint32_t max_bn, pair_min_m;
    int pair;
    uint32_t pair_single_tile, x_ring_bytes, max_x_stages, max_w_stages, grid, raster_gm, no_dp, no_pdl, acc_stages, host_chunk_m,
        host_chunks, no_quad, auto_tile;
};
Knobs knobs() {
    auto g = [](TuneId i) { return g_tune[i].load(std::memory_order_relaxed); };
    Knobs k;
    k.max_bn = uint32_t(g(kTuneMaxBN));
    k.pair_min_m = uint32_t(g(kTunePairMinM));
    k.pair = int(g(kTunePair));
    k.pair_single_tile = uint32_t(g(kTunePairSingleTile));
    k.x_ring_bytes = uint32_t(g(kTuneXRingBytes));
    k.max_x_stages = uint32_t(g(kTuneMaxXStages));
    k.max_w_stages = uint32_t(g(kTuneMaxWStages));
    k.grid = uint32_t(g(kTuneGrid));
    k.raster_gm = uint32_t(g(kTuneRasterGM));
    k.no_dp = uint32_t(g(kTuneNoDP));
    k.no_pdl = uint32_t(g(kTuneNoPDL));
    k.acc_stages = uint32_t(g(kTuneAccStages));
    k.host_chunk_m = uint32_t(g(kTuneHostChunkM));
    k.host_chunks = uint32_t(g(kTuneHostChunks));
    k.no_quad = uint32_t(g(kTuneNoQuad));
    k.auto_tile = uint32_t(g(kTuneAutoTile));
    return k;
}

uint32_t choose_bn(uint32_t m, uint32_t cap, uint32_t* mt) {
    const uint32_t MT = (m + cap - 1) / cap;
    const uint32_t per = (m + MT - 1) / MT;
    *mt = MT;
    return std::max(16u, (per + 15) / 16 * 16);
}

// Token-tile cap and CTA-pair policy for a single GEMM under the default
// knobs (auto_tile). The base rule (fewest token tiles of <= 192 tokens,
// pairs from pair_min_m tokens) is tuned on the LLaMA-2-70B shapes; three
// measured corrections for GEMMs with few weight tiles or a short k
// (tools/sched_sweep.py on B200, every variant bit-identical):
//  A  k < 32 k-blocks and >= 2 rounds of pair tiles: no pairs. With 16
//     k-blocks per tile the pair kernel's per-tile cost shows (LLaMA-2-7B
//     gate_up M = 256 / 512 / 1024: 32.4 -> 30.6, 53.3 -> 48.5,
//     91.4 -> 85.8 us; qkv M = 1024 56.3 -> 51.5 us).
//  B  one round of whole pair tiles that leaves units idle (T <= U < 2T,
//     no split): more, smaller token tiles while they still fit in one round
//     and stay >= 128 tokens (7B o M = 512 15.1 -> 13.4 us, down M = 512
//     27.3 -> 23.5 us).
//  C  split tiles (2T <= U: halves or equal pieces): halve the token tile
//     instead, if each CTA's weight stream of the 2T smaller tiles stays
//     within the equal-piece bound -- short k streams its whole tile faster
//     than a split reduces (7B o M = 256 13.4 -> 11.5 us, down M = 128
//     17.9 -> 17.1 us; not for down at M = 256, whose 43 k-blocks per tile
//     stream 731 KB per CTA: 19.5 -> 24.7 us measured).
// Returns the token-tile cap and sets *pair_pol (-1 auto, 0 never).
uint32_t pick_tiles(const ImageGeom& G, uint32_t m, uint32_t num_sms, uint32_t pair_min_m, int* pair_pol) {
    constexpr uint64_t kPieceBytes = 400u * 1024u;  // the equal-piece bound of launch_core
    // D  small weights (<= 12 MB, e.g. 7B o 4096 x 4096) at 33-128 tokens:
    //    32-token one-CTA tiles -- the cheap sentinel split-K and MT passes
    //    over L2-resident weights beat a few large split tiles (7B o M = 64 /
    //    96 / 128: 11.3 -> 8.4, 12.4 -> 9.1, 11.2 -> 9.4 us; 7B down, 23 MB,
    //    measured slower at M >= 96, so the bound).
    if (m > 32 && m <= 128 && uint64_t(G.NT) * G.KB * G.chunk_bytes <= (12ull << 20)) {
        *pair_pol = 0;
        return 32;
    }
    uint32_t mt;
    const uint32_t bn = choose_bn(m, kMaxTileM, &mt);
    const uint32_t units_np = std::min<uint32_t>(num_sms, kMaxSlots), units_p = units_np / 2;
    if (m < pair_min_m || G.NT % 2 != 0 || units_p < 1) return kMaxTileM;
    const uint32_t ntp = G.NT / 2;
    auto pair_bn = [&](uint32_t t) {
        uint32_t x;
        const uint32_t b = choose_bn((m + t - 1) / t, kMaxTileM, &x);
        return std::min(kMaxTileM, (b + 31) / 32 * 32);
    };
    const uint64_t T = uint64_t(ntp) * mt;
    if (G.KB < 32 && T >= 2ull * units_p) {  // A
        *pair_pol = 0;
        return kMaxTileM;
    }
    const uint32_t bnp = std::min(kMaxTileM, (bn + 31) / 32 * 32);
    if (bnp < 128) return kMaxTileM;
    if (T <= units_p && 2 * T > units_p) {  // B
        uint32_t best = 0;
        for (uint32_t t = mt + 1; t <= 4 * mt; ++t) {
            if (pair_bn(t) < 128 || uint64_t(ntp) * t > units_p) break;
            best = t;
        }
        return best ? pair_bn(best) : kMaxTileM;
    }
    if (2 * T <= units_p) {  // C
        const uint32_t t = 2 * mt, b = pair_bn(t);
        const uint64_t T2 = uint64_t(ntp) * t;
        const uint64_t pp = T2 ? units_p / T2 : 0;
        if (pp >= 1 && uint64_t(G.KB) * G.chunk_bytes / pp <= kPieceBytes) return b;
    }
    return kMaxTileM;
}

// Activation tensor maps, cached per thread: encoding one costs ~1 us of host
// time, which matters for eager decode GEMMs of a few microseconds. The key
// is everything the map encodes.
struct TmapKey {
    const void* ptr;
    uint64_t k, m, ldx;
    uint32_t box_rows;
    bool operator==(const TmapKey& o) const {
        return ptr == o.ptr && k == o.k && m == o.m && ldx == o.ldx && box_rows == o.box_rows;
    }
};

int activation_tmap(const int8_t* d_x, uint32_t k, uint32_t m, int64_t ldx, uint32_t box_rows, CUtensorMap* out) {
    constexpr int kCache = 16;
    struct Entry {
        TmapKey key;
        CUtensorMap map;
        bool used;
    };
    static thread_local Entry cache[kCache];
    static thread_local int next = 0;
    const TmapKey key{d_x, k, m, uint64_t(ldx), box_rows};
    for (const Entry& e : cache)
        if (e.used && e.key == key) {
            *out = e.map;
            return LQG_OK;
        }
    EncodeTiledFn enc = encode_fn();
    if (!enc) return set_err(LQG_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {k, m};
    const cuuint64_t strides[1] = {cuuint64_t(ldx)};
    const cuuint32_t box[2] = {kXAtom, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(d_x), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS)
        return set_err(LQG_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(cr)) + ")");
    Entry& e = cache[next];
    next = (next + 1) % kCache;
    e.key = key;
    e.map = *out;
    e.used = true;
    return LQG_OK;
}

// Co-resident 2-CTA (or 4-CTA) clusters for the pair kernel at this
// shared-memory size (not every SM can host part of a cluster: GPC / TPC
// boundaries), per device.
int pair_clusters(int device, size_t smem, uint32_t grid, uint32_t cluster = 2) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, size_t>, int>> memo;
    const size_t key = smem * 8 + cluster;
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : memo)
        if (e.first.first == device && e.first.second == key) return e.second;
    const int nc = pair_clusters_kind3(smem, grid, cluster);
    memo.push_back({{device, key}, nc});
    return nc;
}

// The kernels of each output kind live in their own translation unit.
constexpr LaunchFn kLaunchByKind[4] = {launch_gemm_kind0, launch_gemm_kind1, launch_gemm_kind2, launch_gemm_kind3};

// One launch over `ng` weight groups sharing n, k and group size (ng == 1: a
// plain GEMM). Group e owns rows [row0_e, row0_e + m[e]) of X, token scales
// and Y, concatenated in group order.
int launch_core(const lqg_weights* const* ws_list, uint32_t ng, const uint32_t* m_list,
                const int8_t* d_x, int64_t ldx, const float* d_ts, void* d_out, int64_t ldo,
                uint32_t out_kind, lqg_workspace* ws, cudaStream_t stream,
                void* const* fan = nullptr, uint32_t n_fan = 0) {
    Knobs K = knobs();
    const lqg_weights* w = ws_list[0];
    const ImageGeom& G = w->geom;
    uint64_t rows = 0;
    uint32_t max_m = 0;
    for (uint32_t e = 0; e < ng; ++e) {
        const lqg_weights* we = ws_list[e];
        if (!we) return set_err(LQG_EVALIDATION, "null handle");
        if (we->geom.n != G.n || we->geom.k != G.k || we->geom.g != G.g || we->device != w->device)
            return set_err(LQG_EVALIDATION, "grouped weights must share n, k, group_size and device");
        rows += m_list[e];
        max_m = std::max(max_m, m_list[e]);
    }
    if (rows < 1) return set_err(LQG_EVALIDATION, "activation dimensions must be >= 1");
    if (rows >= (uint64_t(1) << 31)) return set_err(LQG_EVALIDATION, "too many activation rows");
    const uint32_t m = static_cast<uint32_t>(rows);
    if (int64_t(G.k) * 127 * 127 >= (int64_t(1) << 31))
        return set_err(LQG_EVALIDATION, "k = " + std::to_string(G.k) +
                                            " risks 32-bit accumulator overflow (k*127*127 >= 2^31)");
    if (!d_x || !d_out || (out_kind != kOutAcc && !d_ts))
        return set_err(LQG_EVALIDATION, "null device pointer");
    if (ldx < int64_t(G.k) || ldx % 16 != 0 || (reinterpret_cast<uintptr_t>(d_x) % 16) != 0)
        return set_err(LQG_EVALIDATION, "activation pitch must be >= k and 16-byte aligned");
    if (ldo < int64_t(G.n)) return set_err(LQG_EVALIDATION, "output pitch must be >= n");
    if (n_fan > 7) return set_err(LQG_EVALIDATION, "at most 8 output destinations");
    for (uint32_t r = 0; r < n_fan; ++r)
        if (!fan[r]) return set_err(LQG_EVALIDATION, "null device pointer");
    if (ws && ws->device != w->device)
        return set_err(LQG_EVALIDATION, "workspace lives on another device");
    lqg_workspace* W = ws;
    if (!W) {
        int rc = default_workspace(w->device, stream, &W);
        if (rc) return rc;
    }

    // Token tile from the largest group; every group gets ceil(m_e / BN) tiles.
    uint32_t MT;
    if (K.auto_tile && ng == 1 && n_fan == 0 && K.max_bn == kMaxTileM && K.pair == -1)
        K.max_bn = pick_tiles(G, max_m, w->num_sms, K.pair_min_m, &K.pair);
    uint32_t BN = choose_bn(max_m, K.max_bn, &MT);
    // CTA pairs (tcgen05 cta_group::2) for multi-token-tile GEMMs: the two
    // CTAs of a cluster own adjacent weight tiles and each loads half of the
    // activation tile, halving the per-SM activation SMEM traffic. The token
    // tile is a multiple of 32 (16 tokens per CTA half). Grouped launches
    // decide on the largest group (its token tiles dominate).
    const bool pair_legal = n_fan == 0 && (MT > 1 || K.pair_single_tile) && G.NT % 2 == 0 && w->num_sms >= 2;
    const bool pair = pair_legal && (K.pair == 1 || (K.pair == -1 && max_m >= K.pair_min_m));
    if (pair) BN = std::min(kMaxTileM, (BN + 31) / 32 * 32);
    CUtensorMap tmap;
    {
        int rc = activation_tmap(d_x, G.k, m, ldx, pair ? BN / 2 : BN, &tmap);
        if (rc) return rc;
    }


    GroupTable<kMaxGroups> gt{};
    uint32_t tiles = 0, row0 = 0;
    for (uint32_t e = 0; e < ng; ++e) {
        GroupEntry& ge = gt.e[e];
        ge.wimg = ws_list[e]->d_img;
        ge.cs = ws_list[e]->d_cs;
        ge.row0 = row0;
        ge.M = m_list[e];
        ge.MT = (m_list[e] + BN - 1) / BN;
        ge.tile0 = tiles;
        tiles += ge.MT * (pair ? G.NT / 2 : G.NT);
        row0 += m_list[e];
    }
    gt.n = ng;

    GemmParams p{};
    p.ts = d_ts;
    p.out = d_out;
    p.ldo = ldo;
    for (uint32_t r = 0; r < n_fan; ++r) p.fan[r] = fan[r];
    p.n_fan = n_fan;
    p.parts = W->parts;
    p.flags = reinterpret_cast<uint32_t*>(W->parts + kMaxSlots * kSlotCells);
    p.N = G.n;
    p.KB = G.KB;
    p.NT = pair ? G.NT / 2 : G.NT;  // scheduling tiles (pair tiles in pair mode)
    p.pair = pair ? 1u : 0u;
    p.MT = MT;  // token tiles of the largest group
    p.tiles = tiles;
    p.BN = BN;
    p.P = G.P;
    p.chunk_bytes = G.chunk_bytes;
    p.out_kind = out_kind;
    p.trace_slot = static_cast<uint32_t>(g_launches.load(std::memory_order_relaxed) % 8);
    // Rings. The TMA engine serves an SM's copies in issue order, so an
    // activation tile issued behind d weight chunks lands only after them:
    // the X ring must run at least as far ahead as the W ring or the MMA
    // stalls on activations (measured: W 12 deep / X 8 deep at decode, W 8 /
    // X 2 at M = 128). Both rings get the same depth, X takes any remaining
    // space.
    p.x_slot_bytes = (pair ? BN / 2 : BN) * kKBlock;
    const uint32_t ring_budget = kSmemMax - kSmemMisc;
    // Decode tiles (<= 32 tokens) keep the W ring at 6: deeper weight
    // prefetch only delays the activation tiles queued behind it (LLaMA-2-70B
    // 4-GEMM step at M = 16: 69 us at 6, 73 us at 10).
    const uint32_t w_cap = BN <= 32 ? kDecodeWStages : kMaxStages;
    // Both rings are EVEN: the two dequant warpgroups take alternate
    // k-blocks and wait on the W (and X) full barriers by parity; with an even
    // ring each warpgroup owns its slots, so the phase before the one it waits
    // for is its own, already consumed. With an odd ring that phase belongs to
    // the other warpgroup, whose TMA may still be in flight: a warpgroup
    // running ahead then sees the parity of the phase two back and reads a
    // slot that has not landed (found by tools/pair_stress.py).
    uint32_t sw = std::min({ring_budget / (p.x_slot_bytes + G.chunk_bytes), K.max_w_stages, w_cap}) & ~1u;
    if (K.x_ring_bytes) sw = std::min(sw, std::max(2u, ((ring_budget - std::min(ring_budget, K.x_ring_bytes)) / G.chunk_bytes) & ~1u));
    p.x_stages = std::min({(ring_budget - sw * G.chunk_bytes) / p.x_slot_bytes, K.max_x_stages, kMaxStages}) & ~1u;
    if (p.x_stages < 2) return set_err(LQG_EVALIDATION, "tile configuration does not fit shared memory");
    p.w_base = p.x_stages * p.x_slot_bytes;
    // A split-K finisher of a large token tile gathers each contributor's
    // whole INT32 partial (BN x 128 x 4 bytes) into the idle rings: they must
    // hold at least one (max_w_stages yields to this).
    if (BN / 16 > kSentinelMaxChunks) {
        const uint32_t need = BN * kTileN * 4;
        while (p.w_base + sw * G.chunk_bytes < need && sw + 2 <= kMaxStages) sw += 2;
        if (p.w_base + sw * G.chunk_bytes < need || p.w_base + sw * G.chunk_bytes > ring_budget)
            return set_err(LQG_EVALIDATION, "tile configuration does not fit shared memory");
    }
    if (sw < 2) return set_err(LQG_EVALIDATION, "tile configuration does not fit shared memory");
    p.w_stages = sw;
    p.acc_stages = K.acc_stages;
    if (tmem_plan(BN, p.acc_stages).a_slots < 2)
        return set_err(LQG_EVALIDATION, "tile configuration does not fit tensor memory");
    const uint64_t total_iters = uint64_t(tiles) * G.KB;
    if (total_iters * kMaxSlots >= (uint64_t(1) << 32))
        return set_err(LQG_EVALIDATION, "problem too large for one launch (tiles x k-blocks x " +
                                            std::to_string(kMaxSlots) + " >= 2^32)");
    uint32_t grid = static_cast<uint32_t>(
        std::min<uint64_t>(std::min<uint32_t>(w->num_sms, kMaxSlots), total_iters));
    if (K.grid) grid = static_cast<uint32_t>(std::min<uint64_t>({K.grid, uint64_t(kMaxSlots), total_iters}));
    // pair mode: scheduling units are CTA pairs (grid = 2 x units)
    uint32_t units = pair ? std::max(1u, grid / 2) : grid;
    const size_t smem = size_t(p.w_base) + size_t(p.w_stages) * G.chunk_bytes + kSmemMisc;

    DeviceGuard dg(w->device);
    if (pair) {
        // size the persistent grid to the clusters that are co-resident, so no
        // pair runs in a second wave
        const int nc = pair_clusters(w->device, smem, 2 * units);
        if (nc > 0 && uint32_t(nc) < units) units = uint32_t(nc);
        grid = 2 * units;
    }
    // Fewer tiles than units, large token tiles: the stream-K split's tail
    // (contributors publish at the end of their ranges, the finisher gathers
    // and stores after them) costs more than idle SMs. Use exactly 2 units per
    // tile (equal halves: every unit one piece, no middle pieces) when they
    // fit, else one unit per tile (no split at all). LLaMA-2-70B on B200:
    // o at M = 128 18.3 -> 17.4 us, qkv at M = 128 19.4 -> 18.6 us, o at
    // M = 256 22.8 -> 19.7 us. Smaller token tiles keep every SM streaming
    // (neutral to +1 % at M = 64, and decode is HBM-bound).
    if (!K.grid && BN >= 128 && tiles <= units) {
        units = 2 * tiles <= units ? 2 * tiles : tiles;
        grid = pair ? 2 * units : units;
    } else if (!K.grid && tiles < units) {
        // Small token tiles (the sentinel split-K): when a few tiles of a
        // small GEMM would be cut into uneven pieces over all SMs, cut every
        // tile into the same number p of equal pieces instead (p * tiles
        // units), as long as that keeps >= 60 % of the units busy and each
        // CTA's weight stream small enough to finish at the per-SM rate.
        // LLaMA-2-7B on B200 at M = 16 / 32: o 7.3 -> 6.1 / 10.2 -> 7.5 us,
        // down 9.3 -> 8.4 / 12.1 -> 9.7, qkv 9.1 -> 8.6 / 10.6 -> 9.1;
        // Mixtral experts 9.7 -> 8.8 / 10.7 -> 9.5; 70B shapes unchanged.
        const uint32_t pp = units / tiles;
        const uint64_t cta_bytes = uint64_t(G.KB) * G.chunk_bytes / pp;
        if (uint64_t(pp) * tiles * 10 >= uint64_t(units) * 6 && cta_bytes <= 400u * 1024u) {
            units = pp * tiles;
            grid = pair ? 2 * units : units;
        }
    }
    // Quad mode: every unit one half of one large token tile in pair mode --
    // the two pairs of a tile form one 4-CTA cluster and the contributor's
    // partial moves to the finisher through DSMEM (when all those clusters
    // are co-resident).
    uint32_t cluster = pair ? 2u : 1u;
    p.quad = 0;
    if (pair && units == 2 * tiles && BN / 16 > kSentinelMaxChunks && G.KB % 2 == 0 && !K.no_quad &&
        pair_clusters(w->device, smem, 2 * units, 4) >= int(tiles)) {
        p.quad = 1;
        cluster = 4;
    }
    // Hybrid schedule: whole-tile rounds first, stream-K over the last G..2G
    // tiles (all tiles when there are fewer than G), tiles rasterized in groups
    // of GM token tiles sized so that the activation and weight slices of one
    // round balance in L2 (GM^2 ~ G * weight bytes per tile / activation bytes).
    {
        const uint64_t T = tiles;
        uint32_t dp = 0;
        if (T >= units && !K.no_dp) dp = static_cast<uint32_t>(T % units == 0 ? T / units : T / units - 1);
        p.dp_rounds = dp;
        const uint64_t sk_total = (T - uint64_t(dp) * units) * G.KB;
        p.sk_q = static_cast<uint32_t>(sk_total / units);
        p.sk_r = static_cast<uint32_t>(sk_total % units);
        const double ratio = double(units) * ((pair ? 2 : 1) * kTileN / 2.0) / double(BN);
        uint32_t gm = static_cast<uint32_t>(std::lround(std::sqrt(ratio)));
        // Activations that fit in L2 many times over (<= 40 MB of the 126 MB):
        // raster over all token tiles, so X stays L2-resident and every weight
        // tile is read from DRAM once (LLaMA-2-70B at M = 4096, ncu: DRAM
        // traffic qkv 233 -> 159 MB, o 158 -> 123, gate_up 739 -> 407 MB, the
        // algorithmic 160 / 135 / 390 MB; down's 117 MB of X thrashes L2 that
        // way: 1083 -> 1485 MB, so it keeps the balance rule).
        if (uint64_t(m) * G.k <= (40ull << 20)) gm = MT;
        if (K.raster_gm) gm = K.raster_gm;
        p.raster_gm = std::max(1u, std::min(gm, MT));
    }
    KernelSpec ks;
    ks.tmap_x = tmap;
    ks.p = p;
    ks.gt = &gt;
    ks.ng = ng;
    ks.pair = pair;
    ks.fan = n_fan > 0;
    ks.pdl = !K.no_pdl;
    ks.cluster = cluster;
    ks.grid = grid;
    ks.smem = smem;
    ks.stream = stream;
    LQG_CUDA(kLaunchByKind[out_kind](ks));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LQG_CUDA(cudaGetLastError());
    return LQG_OK;
}

int launch_gemm(const lqg_weights* w, const int8_t* d_x, int64_t ldx, const float* d_ts, uint32_t m,
                void* d_out, int64_t ldo, uint32_t out_kind, lqg_workspace* ws, cudaStream_t stream) {
    if (m < 1) return set_err(LQG_EVALIDATION, "activation dimensions must be >= 1");
    return launch_core(&w, 1, &m, d_x, ldx, d_ts, d_out, ldo, out_kind, ws, stream);
}

int ensure_cap(void** ptr, size_t* cap, size_t need) {
    if (*cap >= need) return LQG_OK;
    cudaFree(*ptr);
    *ptr = nullptr;
    *cap = 0;
    if (cudaMalloc(ptr, need) != cudaSuccess) return set_err(LQG_ECUDA, "staging allocation failed");
    *cap = need;
    return LQG_OK;
}

size_t out_elem_bytes(int y_dtype) { return y_dtype == LQG_Y_F32 ? 4 : 2; }

int out_kind_of(int y_dtype, uint32_t* kind) {
    switch (y_dtype) {
        case LQG_Y_F32: *kind = kOutF32; return LQG_OK;
        case LQG_Y_F16: *kind = kOutF16; return LQG_OK;
        case LQG_Y_BF16: *kind = kOutBF16; return LQG_OK;
    }
    return set_err(LQG_EVALIDATION, "unknown output dtype " + std::to_string(y_dtype));
}

}  // namespace

extern "C" {

const char* lqg_last_error(void) { return g_err.c_str(); }

#ifdef LQG_TRACE
// Debug build only: copy the per-CTA %globaltimer trace (160 x 16 u64).
int lqg_debug_trace(unsigned long long* out) {
    // each kernel unit (output kind) has its own trace buffer: merge them
    constexpr size_t kN = 8 * 160 * 16;
    std::vector<unsigned long long> buf(kN);
    std::fill(out, out + kN, 0ull);
    int (*const fns[4])(unsigned long long*) = {debug_trace_kind0, debug_trace_kind1, debug_trace_kind2,
                                                debug_trace_kind3};
    for (auto fn : fns) {
        if (fn(buf.data())) return 4;
        for (size_t i = 0; i < kN; ++i) out[i] = std::max(out[i], buf[i]);
    }
    return 0;
}
#endif
const char* lqg_version(void) { return "lqg 0.1 (sm_100a, tcgen05 kind::i8, TMEM-A LiquidQuant mainloop)"; }
uint64_t lqg_kernel_launch_count(void) { return g_launches.load(); }

int lqg_tune_set(const char* name, int64_t value) {
    if (!name) return set_err(LQG_EVALIDATION, "null argument");
    for (int i = 0; i < kTuneCount; ++i)
        if (std::strcmp(name, kTuneDefs[i].name) == 0) {
            if (value < kTuneDefs[i].lo || value > kTuneDefs[i].hi)
                return set_err(LQG_EVALIDATION, std::string("tune value out of range for ") + name);
            g_tune[i].store(value, std::memory_order_relaxed);
            return LQG_OK;
        }
    return set_err(LQG_EVALIDATION, std::string("unknown tune knob ") + name);
}

int lqg_tune_get(const char* name, int64_t* value) {
    if (!name || !value) return set_err(LQG_EVALIDATION, "null argument");
    for (int i = 0; i < kTuneCount; ++i)
        if (std::strcmp(name, kTuneDefs[i].name) == 0) {
            *value = g_tune[i].load(std::memory_order_relaxed);
            return LQG_OK;
        }
    return set_err(LQG_EVALIDATION, std::string("unknown tune knob ") + name);
}

void lqg_tune_reset(void) {
    for (int i = 0; i < kTuneCount; ++i) g_tune[i].store(kTuneDefs[i].dflt, std::memory_order_relaxed);
}

int lqg_bundle_validate(const lqg_bundle_view* bundle) {
    if (!bundle) return set_err(LQG_EVALIDATION, "null argument");
    return validate_bundle(*bundle);
}

uint64_t lqg_image_bytes(uint32_t n, uint32_t k, uint32_t group_size) {
    if (n < 1 || k < 1 || group_size < 1 || group_size % 32 != 0) return 0;
    const ImageGeom G = make_geom(n, k, group_size);
    return uint64_t(G.NT) * G.KB * G.chunk_bytes;
}

int lqg_prepack_host(const lqg_bundle_view* bundle, uint8_t* image, uint64_t image_bytes) {
    if (!bundle || !image) return set_err(LQG_EVALIDATION, "null argument");
    int rc = validate_bundle(*bundle);
    if (rc) return rc;
    rc = device_layout_supported(bundle->group_size);
    if (rc) return rc;
    const ImageGeom G = make_geom(bundle->n, bundle->k, bundle->group_size);
    if (image_bytes != uint64_t(G.NT) * G.KB * G.chunk_bytes)
        return set_err(LQG_EVALIDATION, "image buffer has wrong size");
    std::vector<uint8_t> img;
    prepack_host(*bundle, G, img);
    std::memcpy(image, img.data(), img.size());
    return LQG_OK;
}

int lqg_weights_from_image(const uint8_t* image, uint64_t image_bytes, const float* channel_scales,
                           uint32_t n, uint32_t k, uint32_t group_size, int device,
                           lqg_weights** out) {
    if (!image || !channel_scales || !out) return set_err(LQG_EVALIDATION, "null argument");
    if (n < 1 || k < 1 || group_size < 1 || k % group_size != 0)
        return set_err(LQG_EVALIDATION, "bad image dimensions");
    int rc = device_layout_supported(group_size);
    if (rc) return rc;
    const ImageGeom G = make_geom(n, k, group_size);
    if (image_bytes != uint64_t(G.NT) * G.KB * G.chunk_bytes)
        return set_err(LQG_EVALIDATION, "image buffer has wrong size");
    for (uint32_t r = 0; r < n; ++r)
        if (!(channel_scales[r] > 0.0f) || !std::isfinite(channel_scales[r]))
            return set_err(LQG_EVALIDATION, "channel scale at row " + std::to_string(r) +
                                                " must be positive and finite");
    lqg_weights* w = nullptr;
    rc = alloc_weights(device, G, &w);
    if (rc) return rc;
    std::vector<float> cs(uint64_t(G.NT) * kTileN, 1.0f);
    std::memcpy(cs.data(), channel_scales, uint64_t(n) * 4);
    DeviceGuard g(device);
    if (cudaMemcpy(w->d_img, image, image_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(w->d_cs, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        lqg_weights_destroy(w);
        return set_err(LQG_ECUDA, "weight upload failed");
    }
    *out = w;
    return LQG_OK;
}

// Plain-layout bundles are prepacked on the device (prepack_plain_kernel):
// the upload is the same n*k/2 + 2*n*k/g bytes as the image, and a 100+ MB
// matrix prepacks in milliseconds instead of a host pass.
static int create_plain_on_device(const lqg_bundle_view& b, const ImageGeom& G, int device,
                                  lqg_weights** out) {
    lqg_weights* w = nullptr;
    int rc = alloc_weights(device, G, &w);
    if (rc) return rc;
    DeviceGuard g(device);
    uint8_t* d_tmp = nullptr;
    const uint64_t ng = b.n_groups;
    const uint64_t tmp_bytes = (b.packed_bytes + 15) / 16 * 16 + 2 * ng;
    if (cudaMalloc(&d_tmp, tmp_bytes) != cudaSuccess) {
        lqg_weights_destroy(w);
        return set_err(LQG_ECUDA, "prepack staging allocation failed");
    }
    uint8_t* d_packed = d_tmp;
    uint8_t* d_scales = d_tmp + (b.packed_bytes + 15) / 16 * 16;
    uint8_t* d_offsets = d_scales + ng;
    std::vector<float> cs(uint64_t(G.NT) * kTileN, 1.0f);
    std::memcpy(cs.data(), b.channel_scales, uint64_t(b.n) * 4);
    cudaError_t e = cudaMemcpy(d_packed, b.packed_weights, b.packed_bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_scales, b.group_scales, ng, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_offsets, b.group_offsets, ng, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(w->d_cs, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        fill_image_kernel<<<1184, 256>>>(w->d_img, uint64_t(G.NT) * G.KB, G.chunk_bytes);
        const uint64_t threads = uint64_t(b.n) * (b.k / 32);
        prepack_plain_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256>>>(
            d_packed, d_scales, d_offsets, b.n, b.k, b.group_size, w->d_img, G.chunk_bytes, G.KB, G.P);
        g_launches.fetch_add(2, std::memory_order_relaxed);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    cudaFree(d_tmp);
    if (e != cudaSuccess) {
        lqg_weights_destroy(w);
        return set_err(LQG_ECUDA, std::string("device prepack failed: ") + cudaGetErrorString(e));
    }
    *out = w;
    return LQG_OK;
}

int lqg_weights_create(const lqg_bundle_view* bundle, int device, lqg_weights** out) {
    if (!bundle || !out) return set_err(LQG_EVALIDATION, "null argument");
    int rc = validate_bundle(*bundle);
    if (rc) return rc;
    rc = device_layout_supported(bundle->group_size);
    if (rc) return rc;
    const ImageGeom G = make_geom(bundle->n, bundle->k, bundle->group_size);
    if (bundle->layout == LQG_LAYOUT_PLAIN) return create_plain_on_device(*bundle, G, device, out);
    std::vector<uint8_t> img;
    prepack_host(*bundle, G, img);
    return lqg_weights_from_image(img.data(), img.size(), bundle->channel_scales, bundle->n,
                                  bundle->k, bundle->group_size, device, out);
}

int lqg_weights_quantize(const float* d_w, int64_t ldw, uint32_t n, uint32_t k, uint32_t group_size,
                         void* stream, lqg_weights** out) {
    if (!d_w || !out) return set_err(LQG_EVALIDATION, "null argument");
    if (n < 1 || k < 1) return set_err(LQG_EVALIDATION, "weight matrix dimensions must be >= 1");
    if (group_size < 1) return set_err(LQG_EVALIDATION, "group_size must be >= 1");
    if (k % group_size != 0)
        return set_err(LQG_EVALIDATION, "k = " + std::to_string(k) + " not divisible by group_size = " +
                                            std::to_string(group_size));
    if (ldw < int64_t(k)) return set_err(LQG_EVALIDATION, "weight pitch must be >= k");
    int rc = device_layout_supported(group_size);
    if (rc) return rc;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, d_w) != cudaSuccess || attr.type != cudaMemoryTypeDevice)
        return set_err(LQG_EVALIDATION, "weights must be a device pointer");
    const ImageGeom G = make_geom(n, k, group_size);
    lqg_weights* w = nullptr;
    rc = alloc_weights(attr.device, G, &w);
    if (rc) return rc;
    DeviceGuard g(attr.device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int8_t* q = nullptr;
    unsigned long long* bad = nullptr;
    auto cleanup = [&] {
        cudaFree(q);
        cudaFree(bad);
    };
    if (cudaMalloc(&q, uint64_t(n) * k) != cudaSuccess || cudaMalloc(&bad, 8) != cudaSuccess) {
        cleanup();
        lqg_weights_destroy(w);
        return set_err(LQG_ECUDA, "quantizer scratch allocation failed");
    }
    cudaMemsetAsync(bad, 0xFF, 8, st);
    {
        const uint64_t nch = uint64_t(G.NT) * G.KB;
        fill_image_kernel<<<1184, 256, 0, st>>>(w->d_img, nch, G.chunk_bytes);
        std::vector<float> ones(uint64_t(G.NT) * kTileN, 1.0f);
        cudaMemcpyAsync(w->d_cs, ones.data(), ones.size() * 4, cudaMemcpyHostToDevice, st);
        quantize_level1_kernel<<<n, 256, 0, st>>>(d_w, ldw, n, k, q, w->d_cs, bad);
        const uint64_t warps = uint64_t(n) * (k / group_size);
        quantize_level2_pack_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(
            q, n, k, group_size, w->d_img, G.chunk_bytes, G.KB, G.P);
        g_launches.fetch_add(3, std::memory_order_relaxed);
    }
    unsigned long long h_bad = 0;
    cudaError_t e = cudaMemcpyAsync(&h_bad, bad, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cleanup();
    if (e != cudaSuccess) {
        lqg_weights_destroy(w);
        return set_err(LQG_ECUDA, std::string("weight quantization failed: ") + cudaGetErrorString(e));
    }
    if (h_bad != ~0ull) {
        lqg_weights_destroy(w);
        return set_err(LQG_EVALIDATION, "non-finite weight at (" + std::to_string(h_bad / k) + ", " +
                                            std::to_string(h_bad % k) + ")");
    }
    *out = w;
    return LQG_OK;
}

int lqg_weights_destroy(lqg_weights* w) {
    if (!w) return LQG_OK;
    DeviceGuard g(w->device);
    cudaFree(w->d_img);
    cudaFree(w->d_cs);
    delete w;
    return LQG_OK;
}

int lqg_weights_shape(const lqg_weights* w, uint32_t* n, uint32_t* k, uint32_t* g) {
    if (!w) return set_err(LQG_EVALIDATION, "null handle");
    if (n) *n = w->geom.n;
    if (k) *k = w->geom.k;
    if (g) *g = w->geom.g;
    return LQG_OK;
}

uint64_t lqg_weights_device_bytes(const lqg_weights* w) {
    return w ? w->img_bytes + uint64_t(w->geom.NT) * kTileN * 4 : 0;
}

// ---------------------------------------------------------------- LQWB files
// The reference's on-disk bundle format (bundle.hpp:5-24; write_bundle /
// read_bundle, bundle.cpp:137-203), all integers little-endian. Errors carry
// the reference's messages; stream failures are LQG_EIO with
// "... (byte offset N)" like lq::IoError (errors.hpp:23-27).
namespace {

struct LqwbReader {
    std::ifstream& in;
    uint64_t off = 0;
    int raw(void* p, uint64_t n) {
        in.read(static_cast<char*>(p), std::streamsize(n));
        if (uint64_t(in.gcount()) != n)
            return set_err(LQG_EIO, "unexpected end of stream (byte offset " + std::to_string(off) + ")");
        off += n;
        return LQG_OK;
    }
    int u16(uint16_t& v) {
        uint8_t b[2];
        int rc = raw(b, 2);
        v = uint16_t(b[0] | (b[1] << 8));
        return rc;
    }
    int u32(uint32_t& v) {
        uint8_t b[4];
        int rc = raw(b, 4);
        v = 0;
        for (int j = 0; j < 4; ++j) v |= uint32_t(b[j]) << (8 * j);
        return rc;
    }
};

struct HostBundle {
    lqg_bundle_view view{};
    std::vector<uint8_t> packed, scales, offsets;
    std::vector<float> cs;
};

// read_bundle (bundle.cpp:168-203) + QuantizedWeightBundle::validate.
int read_lqwb(const char* path, HostBundle& hb) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return set_err(LQG_EIO, std::string("cannot open ") + path + " (byte offset 0)");
    f.seekg(0, std::ios::end);
    const uint64_t fsize = uint64_t(f.tellg());
    f.seekg(0, std::ios::beg);
    LqwbReader r{f};
    char magic[4];
    int rc = r.raw(magic, 4);
    if (rc) return rc;
    if (std::memcmp(magic, "LQWB", 4) != 0) return set_err(LQG_EVALIDATION, "bad magic (not an LQWB file)");
    uint16_t ver;
    if ((rc = r.u16(ver))) return rc;
    if (ver != 1) return set_err(LQG_EVALIDATION, "unsupported version " + std::to_string(ver));
    lqg_bundle_view& b = hb.view;
    if ((rc = r.u32(b.n)) || (rc = r.u32(b.k)) || (rc = r.u32(b.group_size))) return rc;
    uint8_t layout;
    if ((rc = r.raw(&layout, 1))) return rc;
    if (layout > 1) return set_err(LQG_EVALIDATION, "unknown layout flag " + std::to_string(layout));
    b.layout = layout;
    b.fragment = lqg_fragment_descriptor{4, 32, 64, 32, 16, 64};
    if (layout == LQG_LAYOUT_DUAL_MMA) {
        auto& d = b.fragment;
        if ((rc = r.raw(&d.warps_per_group, 1)) || (rc = r.raw(&d.threads_per_warp, 1)) ||
            (rc = r.u16(d.mma_m)) || (rc = r.u16(d.mma_k)) ||
            (rc = r.u16(d.elements_per_thread_per_mma)) || (rc = r.u16(d.dual_k_span)))
            return rc;
    }
    if (b.n < 1 || b.k < 1) return set_err(LQG_EVALIDATION, "bundle dimensions must be >= 1");
    if (b.group_size < 1 || b.k % b.group_size != 0)
        return set_err(LQG_EVALIDATION, "k not divisible by group_size");
    const uint64_t nk = uint64_t(b.n) * b.k;
    const uint64_t ng = uint64_t(b.n) * (b.k / b.group_size);
    // A truncated file fails at the first read that runs past its end, with
    // that read's start offset -- decided before allocating the payload.
    const uint64_t reads[3] = {(nk + 1) / 2, ng, ng};
    uint64_t at = r.off;
    for (uint64_t len : reads) {
        if (at + len > fsize) return set_err(LQG_EIO, "unexpected end of stream (byte offset " + std::to_string(at) + ")");
        at += len;
    }
    if (at + 4ull * b.n > fsize)
        return set_err(LQG_EIO, "unexpected end of stream (byte offset " +
                                    std::to_string(at + (fsize - at) / 4 * 4) + ")");
    hb.packed.resize(reads[0]);
    hb.scales.resize(ng);
    hb.offsets.resize(ng);
    hb.cs.resize(b.n);
    if ((rc = r.raw(hb.packed.data(), reads[0])) || (rc = r.raw(hb.scales.data(), ng)) ||
        (rc = r.raw(hb.offsets.data(), ng)))
        return rc;
    for (uint32_t i = 0; i < b.n; ++i) {
        uint32_t bits;
        if ((rc = r.u32(bits))) return rc;
        std::memcpy(&hb.cs[i], &bits, 4);
    }
    if (r.off != fsize) return set_err(LQG_EVALIDATION, "trailing bytes after payload");
    b.packed_weights = hb.packed.data();
    b.packed_bytes = hb.packed.size();
    b.group_scales = hb.scales.data();
    b.group_offsets = hb.offsets.data();
    b.n_groups = ng;
    b.channel_scales = hb.cs.data();
    return validate_bundle(b);
}

}  // namespace

int lqg_bundle_file_validate(const char* path) {
    if (!path) return set_err(LQG_EVALIDATION, "null argument");
    HostBundle hb;
    return read_lqwb(path, hb);
}

int lqg_weights_load(const char* path, int device, lqg_weights** out) {
    if (!path || !out) return set_err(LQG_EVALIDATION, "null argument");
    HostBundle hb;
    int rc = read_lqwb(path, hb);
    if (rc) return rc;
    return lqg_weights_create(&hb.view, device, out);
}

// write_bundle (bundle.cpp:137-166) of the handle as a PlainRowMajor bundle.
int lqg_weights_save(const lqg_weights* w, const char* path) {
    if (!w || !path) return set_err(LQG_EVALIDATION, "null argument");
    const ImageGeom& G = w->geom;
    const uint64_t nk = uint64_t(G.n) * G.k, ng = uint64_t(G.n) * (G.k / G.g);
    std::vector<uint8_t> packed((nk + 1) / 2, 0), scales(ng), offsets(ng);
    std::vector<float> cs(G.n);
    int rc = lqg_weights_export(w, packed.data(), scales.data(), offsets.data(), cs.data());
    if (rc) return rc;
    std::ofstream f(path, std::ios::binary);
    if (!f) return set_err(LQG_EIO, std::string("cannot open ") + path + " for writing (byte offset 0)");
    std::vector<uint8_t> hdr;
    auto put = [&](uint64_t v, int nbytes) {
        for (int i = 0; i < nbytes; ++i) hdr.push_back(uint8_t(v >> (8 * i)));
    };
    hdr.insert(hdr.end(), {'L', 'Q', 'W', 'B'});
    put(1, 2);
    put(G.n, 4);
    put(G.k, 4);
    put(G.g, 4);
    put(LQG_LAYOUT_PLAIN, 1);
    uint64_t off = 0;
    auto wr = [&](const void* p, uint64_t n) -> int {
        f.write(static_cast<const char*>(p), std::streamsize(n));
        if (!f) return set_err(LQG_EIO, "write failed (byte offset " + std::to_string(off) + ")");
        off += n;
        return LQG_OK;
    };
    std::vector<uint8_t> csb(uint64_t(G.n) * 4);
    for (uint32_t i = 0; i < G.n; ++i) {
        uint32_t bits;
        std::memcpy(&bits, &cs[i], 4);
        for (int j = 0; j < 4; ++j) csb[4 * i + j] = uint8_t(bits >> (8 * j));
    }
    if ((rc = wr(hdr.data(), hdr.size())) || (rc = wr(packed.data(), packed.size())) ||
        (rc = wr(scales.data(), ng)) || (rc = wr(offsets.data(), ng)) || (rc = wr(csb.data(), csb.size())))
        return rc;
    f.flush();
    if (!f) return set_err(LQG_EIO, "flush failed (byte offset " + std::to_string(off) + ")");
    return LQG_OK;
}

int lqg_weights_export(const lqg_weights* w, uint8_t* packed, uint8_t* scales, uint8_t* offsets,
                       float* cs) {
    if (!w) return set_err(LQG_EVALIDATION, "null handle");
    const ImageGeom& G = w->geom;
    std::vector<uint8_t> img(w->img_bytes);
    DeviceGuard g(w->device);
    LQG_CUDA(cudaMemcpy(img.data(), w->d_img, img.size(), cudaMemcpyDeviceToHost));
    if (cs) LQG_CUDA(cudaMemcpy(cs, w->d_cs, uint64_t(G.n) * 4, cudaMemcpyDeviceToHost));
    const uint32_t gpr = G.k / G.g;
    for (uint32_t row = 0; row < G.n; ++row) {
        if (packed) {
            for (uint32_t k0 = 0; k0 < G.k; k0 += 8) {
                const uint32_t kb = k0 / kKBlock, c = (k0 % kKBlock) / 32, wsub = (k0 % 32) / 8;
                uint32_t word;
                std::memcpy(&word, img.data() + code_offset(G.chunk_bytes, G.KB, row, kb, c) + wsub * 4, 4);
                for (uint32_t e = 0; e < 8 && k0 + e < G.k; ++e) {
                    const uint32_t code = (word >> (8 * (e % 4) + 4 * (e / 4))) & 0xF;
                    const uint64_t idx = uint64_t(row) * G.k + k0 + e;
                    if (idx % 2 == 0)
                        packed[idx / 2] = uint8_t((packed[idx / 2] & 0xF0) | code);
                    else
                        packed[idx / 2] = uint8_t((packed[idx / 2] & 0x0F) | (code << 4));
                }
            }
        }
        for (uint32_t gi = 0; gi < gpr; ++gi) {
            const uint32_t k0 = gi * G.g;
            const uint32_t kb = k0 / kKBlock, c = (k0 % kKBlock) / 32;
            const uint8_t* p = img.data() + param_offset(G.chunk_bytes, G.KB, row, kb, c / (kSubBlocks / G.P));
            if (scales) scales[uint64_t(row) * gpr + gi] = p[0];
            if (offsets) offsets[uint64_t(row) * gpr + gi] = p[1];
        }
    }
    return LQG_OK;
}

int lqg_workspace_create(int device, lqg_workspace** out) {
    if (!out) return set_err(LQG_EVALIDATION, "null argument");
    int rc = check_device(device, nullptr);
    if (rc) return rc;
    return workspace_create(device, out);
}

int lqg_workspace_destroy(lqg_workspace* ws) {
    if (!ws) return LQG_OK;
    DeviceGuard g(ws->device);
    cudaFree(ws->parts);
    delete ws;
    return LQG_OK;
}

int lqg_gemm_w4a8(const lqg_weights* w, const int8_t* d_x, int64_t ldx, const float* d_ts, uint32_t m,
                  void* d_y, int64_t ldy, int y_dtype, lqg_workspace* ws, void* stream) {
    if (!w) return set_err(LQG_EVALIDATION, "null handle");
    uint32_t kind;
    int rc = out_kind_of(y_dtype, &kind);
    if (rc) return rc;
    return launch_gemm(w, d_x, ldx, d_ts, m, d_y, ldy, kind, ws, static_cast<cudaStream_t>(stream));
}

int lqg_gemm_w4a8_grouped(const lqg_weights* const* weights, uint32_t num_groups, const int8_t* d_x,
                          int64_t ldx, const float* d_token_scales, const uint32_t* m, void* d_y,
                          int64_t ldy, int y_dtype, lqg_workspace* ws, void* stream) {
    if (!weights || !m) return set_err(LQG_EVALIDATION, "null argument");
    if (num_groups < 1 || num_groups > kMaxGroups)
        return set_err(LQG_EVALIDATION, "num_groups must be in [1, " + std::to_string(kMaxGroups) + "]");
    uint32_t kind;
    int rc = out_kind_of(y_dtype, &kind);
    if (rc) return rc;
    return launch_core(weights, num_groups, m, d_x, ldx, d_token_scales, d_y, ldy, kind, ws,
                       static_cast<cudaStream_t>(stream));
}

int lqg_gemm_w4a8_grouped_accum(const lqg_weights* const* weights, uint32_t num_groups,
                                const int8_t* d_x, int64_t ldx, const uint32_t* m, int32_t* d_acc,
                                int64_t ldacc, lqg_workspace* ws, void* stream) {
    if (!weights || !m) return set_err(LQG_EVALIDATION, "null argument");
    if (num_groups < 1 || num_groups > kMaxGroups)
        return set_err(LQG_EVALIDATION, "num_groups must be in [1, " + std::to_string(kMaxGroups) + "]");
    return launch_core(weights, num_groups, m, d_x, ldx, nullptr, d_acc, ldacc, kOutAcc, ws,
                       static_cast<cudaStream_t>(stream));
}

int lqg_gemm_w4a8_fanout(const lqg_weights* w, const int8_t* d_x, int64_t ldx,
                         const float* d_token_scales, uint32_t m, void* const* d_ys, uint32_t n_ys,
                         int64_t ldy, int y_dtype, lqg_workspace* ws, void* stream) {
    if (!w || !d_ys) return set_err(LQG_EVALIDATION, "null argument");
    if (n_ys < 1 || n_ys > 8) return set_err(LQG_EVALIDATION, "n_ys must be in [1, 8]");
    if (m < 1) return set_err(LQG_EVALIDATION, "activation dimensions must be >= 1");
    uint32_t kind;
    int rc = out_kind_of(y_dtype, &kind);
    if (rc) return rc;
    return launch_core(&w, 1, &m, d_x, ldx, d_token_scales, d_ys[0], ldy, kind, ws,
                       static_cast<cudaStream_t>(stream), d_ys + 1, n_ys - 1);
}

int lqg_gemm_w4a8_accum(const lqg_weights* w, const int8_t* d_x, int64_t ldx, uint32_t m, int32_t* d_acc,
                        int64_t ldacc, lqg_workspace* ws, void* stream) {
    if (!w) return set_err(LQG_EVALIDATION, "null handle");
    return launch_gemm(w, d_x, ldx, nullptr, m, d_acc, ldacc, kOutAcc, ws,
                       static_cast<cudaStream_t>(stream));
}

namespace {

// Device staging of one host-buffer call: X / token-scale / Y buffers, the
// copy-in and copy-out streams and the per-chunk events. Staging contexts live
// in a process-wide pool; each call holds one exclusively, so concurrent host
// threads (on one handle or several) never share buffers, and the weight
// handle itself stays immutable.
struct Staging {
    int device = -1;
    bool busy = false;
    int8_t* d_x = nullptr;
    size_t x_cap = 0;
    float* d_ts = nullptr;
    size_t ts_cap = 0;
    void* d_y = nullptr;
    size_t y_cap = 0;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev[2 * 8 + 1] = {};
};

std::mutex g_staging_mu;
std::vector<Staging*>* g_staging = new std::vector<Staging*>();  // process lifetime

Staging* staging_acquire(int device) {
    std::lock_guard<std::mutex> lk(g_staging_mu);
    for (Staging* s : *g_staging)
        if (!s->busy && s->device == device) {
            s->busy = true;
            return s;
        }
    auto* s = new Staging();
    s->device = device;
    s->busy = true;
    g_staging->push_back(s);
    return s;
}

void staging_release(Staging* s) {
    std::lock_guard<std::mutex> lk(g_staging_mu);
    s->busy = false;
}

int host_call_on(const lqg_weights* w, Staging& S, const int8_t* x, const float* ts, uint32_t m, void* y,
                 uint32_t kind, size_t ebytes, cudaStream_t st) {
    const ImageGeom& G = w->geom;
    const int64_t ldx = (int64_t(G.k) + 15) / 16 * 16;
    int rc = ensure_cap(reinterpret_cast<void**>(&S.d_x), &S.x_cap, size_t(m) * ldx);
    if (!rc) rc = ensure_cap(reinterpret_cast<void**>(&S.d_ts), &S.ts_cap, size_t(m) * 4);
    if (!rc) rc = ensure_cap(&S.d_y, &S.y_cap, size_t(m) * G.n * ebytes);
    if (rc) return rc;
    // Calls of >= host_chunk_m rows are cut into row chunks pipelined over
    // three streams: H2D of chunk c+1 and D2H of chunk c-1 (PCIe is full
    // duplex) overlap the GEMM of chunk c, so the call costs ~max(H2D, D2H)
    // instead of their sum plus the GEMM. Small calls (latency-bound) stay one
    // chunk. B200 box: pinned D2H 55.8 GB/s, H2D + D2H concurrently 87 GB/s;
    // the 70B e2e step (52 calls) 26.1 ms at (2048 rows, 8 chunks) -> 24.3 ms
    // at (384, 6), against a ~17-21 ms PCIe floor (tools/e2e_probe.py).
    const Knobs K = knobs();
    const uint32_t per = m >= K.host_chunk_m ? std::max<uint32_t>(std::min<uint32_t>(1024, K.host_chunk_m / 2),
                                                                   (m + K.host_chunks - 1) / K.host_chunks)
                                             : m;
    const uint32_t nchunk = (m + per - 1) / per;
    if (nchunk > 1 && !S.s_in) {
        LQG_CUDA(cudaStreamCreateWithFlags(&S.s_in, cudaStreamNonBlocking));
        LQG_CUDA(cudaStreamCreateWithFlags(&S.s_out, cudaStreamNonBlocking));
        for (cudaEvent_t& e : S.ev) LQG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaStream_t s_in = nchunk > 1 ? S.s_in : st, s_out = nchunk > 1 ? S.s_out : st;
    if (nchunk > 1) {  // the copies start after the caller's prior work on st
        LQG_CUDA(cudaEventRecord(S.ev[16], st));
        LQG_CUDA(cudaStreamWaitEvent(s_in, S.ev[16], 0));
        LQG_CUDA(cudaStreamWaitEvent(s_out, S.ev[16], 0));
    }
    const size_t yrow = size_t(G.n) * ebytes;
    for (uint32_t c = 0; c < nchunk; ++c) {
        const uint32_t r0 = c * per, rows = std::min(per, m - r0);
        int8_t* dx = S.d_x + size_t(r0) * ldx;
        if (ldx == int64_t(G.k)) {
            LQG_CUDA(cudaMemcpyAsync(dx, x + size_t(r0) * G.k, size_t(rows) * G.k, cudaMemcpyHostToDevice, s_in));
        } else {
            LQG_CUDA(cudaMemcpy2DAsync(dx, ldx, x + size_t(r0) * G.k, G.k, G.k, rows,
                                       cudaMemcpyHostToDevice, s_in));
        }
        if (kind != kOutAcc)
            LQG_CUDA(cudaMemcpyAsync(S.d_ts + r0, ts + r0, size_t(rows) * 4, cudaMemcpyHostToDevice, s_in));
        if (nchunk > 1) {
            LQG_CUDA(cudaEventRecord(S.ev[2 * (c % 8)], s_in));
            LQG_CUDA(cudaStreamWaitEvent(st, S.ev[2 * (c % 8)], 0));
        }
        rc = launch_gemm(w, dx, ldx, S.d_ts + r0, rows, static_cast<uint8_t*>(S.d_y) + r0 * yrow, G.n,
                         kind, nullptr, st);
        if (rc) return rc;
        if (nchunk > 1) {
            LQG_CUDA(cudaEventRecord(S.ev[2 * (c % 8) + 1], st));
            LQG_CUDA(cudaStreamWaitEvent(s_out, S.ev[2 * (c % 8) + 1], 0));
        }
        LQG_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(y) + r0 * yrow,
                                 static_cast<uint8_t*>(S.d_y) + r0 * yrow, rows * yrow,
                                 cudaMemcpyDeviceToHost, s_out));
    }
    LQG_CUDA(cudaStreamSynchronize(s_out));
    if (nchunk > 1) LQG_CUDA(cudaStreamSynchronize(st));
    return LQG_OK;
}

}  // namespace

// Synchronous host-buffer call (the reference's calling convention).
// Re-entrant: each call holds its own staging context from the pool.
static int host_call(const lqg_weights* w, const int8_t* x, const float* ts, uint32_t m, void* y,
                     uint32_t kind, size_t ebytes, cudaStream_t st) {
    if (!w) return set_err(LQG_EVALIDATION, "null handle");
    if (m < 1) return set_err(LQG_EVALIDATION, "activation dimensions must be >= 1");
    if (!x || !y || (kind != kOutAcc && !ts)) return set_err(LQG_EVALIDATION, "null host pointer");
    DeviceGuard g(w->device);
    Staging* S = staging_acquire(w->device);
    const int rc = host_call_on(w, *S, x, ts, m, y, kind, ebytes, st);
    staging_release(S);
    return rc;
}

int lqg_gemm_w4a8_host(const lqg_weights* w, const int8_t* x, const float* ts, uint32_t m, void* y,
                       int y_dtype, void* stream) {
    uint32_t kind;
    int rc = out_kind_of(y_dtype, &kind);
    if (rc) return rc;
    return host_call(w, x, ts, m, y, kind, out_elem_bytes(y_dtype), static_cast<cudaStream_t>(stream));
}

int lqg_gemm_w4a8_accum_host(const lqg_weights* w, const int8_t* x, uint32_t m, int32_t* acc,
                             void* stream) {
    return host_call(w, x, nullptr, m, acc, kOutAcc, 4, static_cast<cudaStream_t>(stream));
}

int lqg_dequant_weights(const lqg_weights* w, int8_t* d_w, int64_t ldw, void* stream) {
    if (!w || !d_w) return set_err(LQG_EVALIDATION, "null argument");
    const ImageGeom& G = w->geom;
    if (ldw < int64_t(G.k)) return set_err(LQG_EVALIDATION, "output pitch must be >= k");
    DeviceGuard g(w->device);
    const uint64_t threads = uint64_t(G.n) * G.KB * kSubBlocks;
    dequant_image_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(w->d_img, G.n, G.k, G.chunk_bytes,
                                                                G.KB, G.P, d_w, ldw);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LQG_CUDA(cudaGetLastError());
    return LQG_OK;
}

int lqg_quantize_activations(const float* d_x, int64_t ldx, uint32_t m, uint32_t k, int8_t* d_q,
                             int64_t ldq, float* d_ts, int check_finite, void* stream) {
    if (m < 1 || k < 1) return set_err(LQG_EVALIDATION, "activation dimensions must be >= 1");
    if (!d_x || !d_q || !d_ts) return set_err(LQG_EVALIDATION, "null device pointer");
    if (ldx < int64_t(k) || ldq < int64_t(k)) return set_err(LQG_EVALIDATION, "pitch must be >= k");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned long long* bad = nullptr;
    if (check_finite) {
        LQG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bad), 8, st));
        LQG_CUDA(cudaMemsetAsync(bad, 0xFF, 8, st));
    }
    quantize_activations_kernel<<<m, 256, 0, st>>>(d_x, ldx, m, k, d_q, ldq, d_ts, bad);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LQG_CUDA(cudaGetLastError());
    if (check_finite) {
        unsigned long long h = 0;
        LQG_CUDA(cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, st));
        LQG_CUDA(cudaFreeAsync(bad, st));
        LQG_CUDA(cudaStreamSynchronize(st));
        if (h != ~0ull)
            return set_err(LQG_EVALIDATION, "non-finite activation at (" + std::to_string(h / k) + ", " +
                                                std::to_string(h % k) + ")");
    }
    return LQG_OK;
}

}  // extern "C"
