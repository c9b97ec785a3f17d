// Drop-in replacement for the reference's W4A8 GEMM entry points
//
//   lq::gemm_w4a8_accum   /root/reference/proj/include/lq/gemm.hpp:49-51
//   lq::gemm_w4a8         /root/reference/proj/include/lq/gemm.hpp:54-55
//
// implemented over the lqg C ABI (include/lqg.h, sm_100a kernels in liblqg.so).
// Same signatures, same validation order and exception types as
// src/gemm.cpp:138-223; the CPU engine is not used. Build recipe: the
// reference's gemm.cpp is compiled with its two GEMM definitions renamed
// (-Dgemm_w4a8_accum=cpu_gemm_w4a8_accum -Dgemm_w4a8=cpu_gemm_w4a8) so its
// remaining functions (TileConfig::validate, quantize_activations_per_token,
// gemm_oracle) are kept, and this file provides the GEMM symbols
// (see INTEGRATION.md and oracle/Makefile target `dropin`).
#include <cstdint>
#include <string>
#include <vector>

#include "lq/gemm.hpp"
#include "lqg.h"

namespace lq {
namespace {

[[noreturn]] void throw_status(int rc) {
    const std::string msg = lqg_last_error();
    switch (rc) {
        case LQG_EVALIDATION: throw ValidationError(msg);
        case LQG_EVERIFICATION: throw VerificationError(msg);
        case LQG_EIO: throw IoError(msg, 0);
        default: throw std::runtime_error("lqg: " + msg);
    }
}

void check(int rc) {
    if (rc != LQG_OK) throw_status(rc);
}

// gemm.cpp:53-57
void check_accumulator_range(std::uint32_t k) {
    if (std::int64_t(k) * 127 * 127 >= (std::int64_t(1) << 31))
        throw ValidationError("k = " + std::to_string(k) +
                              " risks 32-bit accumulator overflow (k*127*127 >= 2^31)");
}

struct DeviceBundle {
    lqg_weights* h = nullptr;
    explicit DeviceBundle(const QuantizedWeightBundle& b) {
        lqg_bundle_view v{};
        v.n = b.n;
        v.k = b.k;
        v.group_size = b.group_size;
        v.layout = b.layout == WeightLayout::DualMmaPacked ? LQG_LAYOUT_DUAL_MMA : LQG_LAYOUT_PLAIN;
        v.fragment = {b.fragment.warps_per_group, b.fragment.threads_per_warp, b.fragment.mma_m,
                      b.fragment.mma_k, b.fragment.elements_per_thread_per_mma,
                      b.fragment.dual_k_span};
        v.packed_weights = b.packed_weights.data();
        v.packed_bytes = b.packed_weights.size();
        v.group_scales = b.group_scales.data();
        v.group_offsets = b.group_offsets.data();
        v.n_groups = b.group_scales.size();
        v.channel_scales = b.channel_scales.data();
        check(lqg_weights_create(&v, 0, &h));
    }
    ~DeviceBundle() { lqg_weights_destroy(h); }
};

// gemm.cpp:141-158: the reference's checks, in its order.
void prepare(const ActivationQuant& act, const QuantizedWeightBundle& weights,
             const TileConfig& tile, Engine engine) {
    weights.validate();
    tile.validate(weights);
    if (act.k != weights.k)
        throw ValidationError("activation depth " + std::to_string(act.k) +
                              " does not match weight depth " + std::to_string(weights.k));
    check_accumulator_range(act.k);
    if (engine == Engine::Packed && tile.k_t % weights.fragment.dual_k_span != 0)
        throw ValidationError("k_t must be a multiple of " +
                              std::to_string(weights.fragment.dual_k_span) +
                              " for the packed engine");
    if (act.values.size() != std::size_t(act.m) * act.k || act.m < 1)
        throw ValidationError("activation buffer size does not match m*k");
}

}  // namespace

std::vector<std::int32_t> gemm_w4a8_accum(const ActivationQuant& act,
                                          const QuantizedWeightBundle& weights,
                                          const TileConfig& tile, Engine engine) {
    prepare(act, weights, tile, engine);
    DeviceBundle dev(weights);
    std::vector<std::int32_t> acc(std::size_t(act.m) * weights.n);
    check(lqg_gemm_w4a8_accum_host(dev.h, act.values.data(), act.m, acc.data(), nullptr));
    return acc;
}

std::vector<float> gemm_w4a8(const ActivationQuant& act, const QuantizedWeightBundle& weights,
                             const TileConfig& tile, Engine engine) {
    prepare(act, weights, tile, engine);
    if (act.token_scales.size() != act.m) throw ValidationError("token scale array has wrong size");
    DeviceBundle dev(weights);
    std::vector<float> y(std::size_t(act.m) * weights.n);
    check(lqg_gemm_w4a8_host(dev.h, act.values.data(), act.token_scales.data(), act.m, y.data(),
                             LQG_Y_F32, nullptr));
    return y;
}

}  // namespace lq
