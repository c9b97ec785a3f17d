// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference CPU library (lqlab, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets
// the Python tests, the golden-vector generator and bench.py's cpu_baseline
// leg call the reference implementation of the W4A8 path directly:
//
//   lq::build_bundle                 quant.cpp:203-232
//   lq::quantize_activations_per_token gemm.cpp:19-47
//   lq::gemm_w4a8_accum / gemm_w4a8  gemm.cpp:138-223
//   lq::gemm_oracle                  gemm.cpp:225-243
//   lq::reconstruct_int8             quant.cpp:234-251
//   lq::to_dual_mma / logical_codes  bundle.cpp:251-274, 227-249
//   lq::save_bundle / load_bundle    bundle.cpp:213-224 (LQWB files)
//
// Status codes follow the reference error taxonomy (errors.hpp:15-28):
// 0 ok, 1 ValidationError, 2 VerificationError, 3 IoError, 9 other.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "lq/bundle.hpp"
#include "lq/cost_model.hpp"
#include "lq/gemm.hpp"
#include "lq/packed.hpp"
#include "lq/quant.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const lq::ValidationError& e) {
        g_err = e.what();
        return 1;
    } catch (const lq::VerificationError& e) {
        g_err = e.what();
        return 2;
    } catch (const lq::IoError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

lq::ActivationQuant make_act(const std::int8_t* q, const float* ts, std::uint32_t m,
                             std::uint32_t k) {
    lq::ActivationQuant a;
    a.m = m;
    a.k = k;
    a.values.assign(q, q + std::size_t(m) * k);
    a.token_scales.assign(ts, ts + m);
    return a;
}

}  // namespace

extern "C" {

const char* lqref_last_error(void) { return g_err.c_str(); }

// Opaque handle = heap QuantizedWeightBundle.
int lqref_bundle_build(const float* w, std::uint32_t n, std::uint32_t k, std::uint32_t g,
                       int layout, void** out) {
    return guarded([&] {
        std::span<const float> ws(w, std::size_t(n) * k);
        auto* b = new lq::QuantizedWeightBundle(lq::build_bundle(
            ws, n, k, g,
            layout ? lq::WeightLayout::DualMmaPacked : lq::WeightLayout::PlainRowMajor));
        *out = b;
    });
}

int lqref_bundle_from_arrays(std::uint32_t n, std::uint32_t k, std::uint32_t g, int layout,
                             const std::uint8_t* packed, std::uint64_t packed_len,
                             const std::uint8_t* scales, const std::uint8_t* offsets,
                             std::uint64_t ngroups, const float* cs, void** out) {
    return guarded([&] {
        auto* b = new lq::QuantizedWeightBundle();
        b->n = n;
        b->k = k;
        b->group_size = g;
        b->layout = layout ? lq::WeightLayout::DualMmaPacked : lq::WeightLayout::PlainRowMajor;
        b->packed_weights.assign(packed, packed + packed_len);
        b->group_scales.assign(scales, scales + ngroups);
        b->group_offsets.assign(offsets, offsets + ngroups);
        b->channel_scales.assign(cs, cs + n);
        *out = b;
    });
}

// lq::load_profile + the closed-form diagnostics (cost_model.cpp:150-170).
int lqref_profile_diag(const char* path, double* m_star, double* alpha_mem, double* alpha_comp_150) {
    return guarded([&] {
        const lq::HardwareProfile p = lq::load_profile(path);
        *m_star = lq::transition_batch(p, 4, 8);
        *alpha_mem = lq::alpha_threshold_memory(p, 4);
        *alpha_comp_150 = lq::alpha_threshold_compute(p, 8, 150.0);
    });
}

// lq::total_time of one W4A8 GEMM (cost_model.cpp:137-148).
int lqref_cost_total(const char* path, std::uint64_t n, std::uint64_t k, std::uint64_t m,
                     std::uint32_t m_t, std::uint32_t n_t, std::uint32_t k_t, double alpha,
                     double* seconds, int* compute_bound) {
    return guarded([&] {
        const lq::HardwareProfile p = lq::load_profile(path);
        lq::CostQuery q;
        q.n = n;
        q.k = k;
        q.tile = lq::TileConfig{m_t, n_t, k_t};
        q.weight_bits = 4;
        q.act_bits = 8;
        q.alpha = alpha;
        q.batch = m;
        const lq::CostBreakdown c = lq::total_time(q, p);
        *seconds = c.total;
        *compute_bound = c.regime == lq::Regime::ComputeBound;
    });
}

int lqref_save_bundle(const void* h, const char* path) {
    return guarded([&] { lq::save_bundle(*static_cast<const lq::QuantizedWeightBundle*>(h), path); });
}

int lqref_load_bundle(const char* path, void** out) {
    return guarded([&] { *out = new lq::QuantizedWeightBundle(lq::load_bundle(path)); });
}

void lqref_bundle_free(void* h) { delete static_cast<lq::QuantizedWeightBundle*>(h); }

int lqref_bundle_info(const void* h, std::uint32_t* n, std::uint32_t* k, std::uint32_t* g,
                      int* layout, std::uint64_t* packed_len, std::uint64_t* ngroups) {
    const auto* b = static_cast<const lq::QuantizedWeightBundle*>(h);
    *n = b->n;
    *k = b->k;
    *g = b->group_size;
    *layout = int(b->layout);
    *packed_len = b->packed_weights.size();
    *ngroups = b->group_scales.size();
    return 0;
}

int lqref_bundle_copy_out(const void* h, std::uint8_t* packed, std::uint8_t* scales,
                          std::uint8_t* offsets, float* cs) {
    const auto* b = static_cast<const lq::QuantizedWeightBundle*>(h);
    if (packed) std::memcpy(packed, b->packed_weights.data(), b->packed_weights.size());
    if (scales) std::memcpy(scales, b->group_scales.data(), b->group_scales.size());
    if (offsets) std::memcpy(offsets, b->group_offsets.data(), b->group_offsets.size());
    if (cs) std::memcpy(cs, b->channel_scales.data(), b->channel_scales.size() * 4);
    return 0;
}

int lqref_bundle_validate(const void* h) {
    return guarded([&] { static_cast<const lq::QuantizedWeightBundle*>(h)->validate(); });
}

int lqref_to_dual(const void* h, void** out) {
    return guarded([&] {
        *out = new lq::QuantizedWeightBundle(
            lq::to_dual_mma(*static_cast<const lq::QuantizedWeightBundle*>(h)));
    });
}

int lqref_to_plain(const void* h, void** out) {
    return guarded([&] {
        *out = new lq::QuantizedWeightBundle(
            lq::to_plain(*static_cast<const lq::QuantizedWeightBundle*>(h)));
    });
}

int lqref_logical_codes(const void* h, std::uint8_t* out) {
    return guarded([&] {
        const auto c = lq::logical_codes(*static_cast<const lq::QuantizedWeightBundle*>(h));
        std::memcpy(out, c.data(), c.size());
    });
}

int lqref_reconstruct_int8(const void* h, std::int8_t* out) {
    return guarded([&] {
        const auto w = lq::reconstruct_int8(*static_cast<const lq::QuantizedWeightBundle*>(h));
        std::memcpy(out, w.data(), w.size());
    });
}

int lqref_quantize_activations(const float* x, std::uint32_t m, std::uint32_t k,
                               std::int8_t* q, float* ts) {
    return guarded([&] {
        const auto a = lq::quantize_activations_per_token(
            std::span<const float>(x, std::size_t(m) * k), m, k);
        std::memcpy(q, a.values.data(), a.values.size());
        std::memcpy(ts, a.token_scales.data(), a.token_scales.size() * 4);
    });
}

int lqref_gemm_w4a8_accum(const void* h, const std::int8_t* q, const float* ts,
                          std::uint32_t m, std::uint32_t k, std::uint32_t mt, std::uint32_t nt,
                          std::uint32_t kt, int engine, std::int32_t* acc) {
    return guarded([&] {
        const auto act = make_act(q, ts, m, k);
        const auto r = lq::gemm_w4a8_accum(act, *static_cast<const lq::QuantizedWeightBundle*>(h),
                                           lq::TileConfig{mt, nt, kt},
                                           engine ? lq::Engine::Packed : lq::Engine::Scalar);
        std::memcpy(acc, r.data(), r.size() * 4);
    });
}

int lqref_gemm_w4a8(const void* h, const std::int8_t* q, const float* ts, std::uint32_t m,
                    std::uint32_t k, std::uint32_t mt, std::uint32_t nt, std::uint32_t kt,
                    int engine, float* y) {
    return guarded([&] {
        const auto act = make_act(q, ts, m, k);
        const auto r = lq::gemm_w4a8(act, *static_cast<const lq::QuantizedWeightBundle*>(h),
                                     lq::TileConfig{mt, nt, kt},
                                     engine ? lq::Engine::Packed : lq::Engine::Scalar);
        std::memcpy(y, r.data(), r.size() * 4);
    });
}

// CPU baseline with host threads (BASELINE.md §3 variant (ii)): one std::thread
// per 64-row-aligned N-shard of a DualMmaPacked bundle, each calling the
// unmodified lq::gemm_w4a8 on its shard (legal: output tiles are independent,
// SPEC.md:446-447). Shards are carved once, outside the timed call, by
// lqref_shard_prepare; lqref_gemm_w4a8_sharded only runs the threads.
struct Shards {
    std::vector<lq::QuantizedWeightBundle> parts;
    std::vector<std::uint32_t> row0;
    std::uint32_t n = 0;
};

int lqref_shard_prepare(const void* h, int nthreads, void** out) {
    return guarded([&] {
        const auto& b = *static_cast<const lq::QuantizedWeightBundle*>(h);
        if (b.layout != lq::WeightLayout::DualMmaPacked)
            throw lq::ValidationError("sharded baseline expects a DualMmaPacked bundle");
        auto* s = new Shards();
        s->n = b.n;
        const std::uint32_t band = b.fragment.mma_m;
        const std::uint32_t bands = b.n / band;
        const std::uint32_t gpr = b.groups_per_row();
        const std::uint64_t band_bytes = std::uint64_t(band) * b.k / 2;
        const std::uint32_t parts = std::max(1u, std::min<std::uint32_t>(nthreads, bands));
        for (std::uint32_t p = 0; p < parts; ++p) {
            const std::uint32_t b0 = bands * p / parts, b1 = bands * (p + 1) / parts;
            if (b1 == b0) continue;
            lq::QuantizedWeightBundle sb;
            sb.n = (b1 - b0) * band;
            sb.k = b.k;
            sb.group_size = b.group_size;
            sb.layout = b.layout;
            sb.fragment = b.fragment;
            sb.packed_weights.assign(b.packed_weights.begin() + b0 * band_bytes,
                                     b.packed_weights.begin() + b1 * band_bytes);
            const std::uint64_t r0 = std::uint64_t(b0) * band, r1 = std::uint64_t(b1) * band;
            sb.group_scales.assign(b.group_scales.begin() + r0 * gpr,
                                   b.group_scales.begin() + r1 * gpr);
            sb.group_offsets.assign(b.group_offsets.begin() + r0 * gpr,
                                    b.group_offsets.begin() + r1 * gpr);
            sb.channel_scales.assign(b.channel_scales.begin() + r0, b.channel_scales.begin() + r1);
            s->parts.push_back(std::move(sb));
            s->row0.push_back(std::uint32_t(r0));
        }
        *out = s;
    });
}

void lqref_shard_free(void* s) { delete static_cast<Shards*>(s); }

int lqref_gemm_w4a8_sharded(const void* sh, const std::int8_t* q, const float* ts,
                            std::uint32_t m, std::uint32_t k, float* y) {
    return guarded([&] {
        const auto& s = *static_cast<const Shards*>(sh);
        const auto act = make_act(q, ts, m, k);
        std::vector<std::vector<float>> outs(s.parts.size());
        std::vector<std::thread> th;
        std::vector<std::exception_ptr> errs(s.parts.size());
        for (std::size_t p = 0; p < s.parts.size(); ++p)
            th.emplace_back([&, p] {
                try {
                    outs[p] = lq::gemm_w4a8(act, s.parts[p], lq::TileConfig{64, 64, 64},
                                            lq::Engine::Packed);
                } catch (...) {
                    errs[p] = std::current_exception();
                }
            });
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        for (std::size_t p = 0; p < s.parts.size(); ++p) {
            const std::uint32_t np = s.parts[p].n;
            for (std::uint32_t i = 0; i < m; ++i)
                std::memcpy(y + std::size_t(i) * s.n + s.row0[p],
                            outs[p].data() + std::size_t(i) * np, std::size_t(np) * 4);
        }
    });
}

int lqref_gemm_oracle(const std::int8_t* q, const float* ts, std::uint32_t m, std::uint32_t k,
                      const std::int8_t* w_i8, const float* cs, std::uint32_t n,
                      std::int64_t* acc, float* y) {
    return guarded([&] {
        const auto act = make_act(q, ts, m, k);
        const auto r = lq::gemm_oracle(act, std::span<const std::int8_t>(w_i8, std::size_t(n) * k),
                                       std::span<const float>(cs, n), n);
        if (acc) std::memcpy(acc, r.accum.data(), r.accum.size() * 8);
        if (y) std::memcpy(y, r.y.data(), r.y.size() * 4);
    });
}

int lqref_dequant_word(std::uint32_t w, std::uint8_t s, std::uint8_t a, std::uint32_t* lo,
                       std::uint32_t* hi) {
    lq::InstructionCounter c;
    const auto [l, h] = lq::dequant_word(lq::RegisterWord{w}, s, a, c);
    *lo = l.value;
    *hi = h.value;
    return int(c.total());
}

}  // extern "C"
