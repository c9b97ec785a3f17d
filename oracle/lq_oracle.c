/* TEST INFRASTRUCTURE ONLY — CPU oracle for the W4A8 LiquidGEMM path.
 * See lq_oracle.h for scope, pinning and the usage rule. Reference paths are
 * relative to /root/reference/proj. */
#include "lq_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}

const char* lqo_last_error(void) { return g_err; }

/* quant.hpp:33-35 */
int lqo_round_half_away(double v) { return (int)(v < 0 ? v - 0.5 : v + 0.5); }

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* quant.cpp:14-44 */
int lqo_quantize_first_level(const float* w, uint32_t n, uint32_t k, int8_t* q, float* cs) {
    if (n < 1 || k < 1) return fail("weight matrix dimensions must be >= 1");
    for (uint32_t i = 0; i < n; ++i) {
        const float* row = w + (uint64_t)i * k;
        float amax = 0.0f;
        for (uint32_t j = 0; j < k; ++j) {
            if (!isfinite(row[j])) {
                snprintf(g_err, sizeof g_err, "non-finite weight at (%u, %u)", i, j);
                return 1;
            }
            const float a = fabsf(row[j]);
            amax = amax < a ? a : amax; /* std::max(amax, a) keeps amax on ties */
        }
        const float s = amax == 0.0f ? 1.0f : amax / 119; /* float / int -> float */
        cs[i] = s;
        for (uint32_t j = 0; j < k; ++j)
            q[(uint64_t)i * k + j] =
                (int8_t)clampi(lqo_round_half_away((double)row[j] / s), -119, 119);
    }
    return 0;
}

/* quant.cpp:48-60 */
static void group_params(int mn, int mx, uint8_t* s_out, uint8_t* a_out) {
    const int span = mx - mn;
    int s = lqo_round_half_away((double)span / 15.0);
    if (s < 1) s = 1;
    *s_out = (uint8_t)s;
    *a_out = (uint8_t)(128 + mn);
}

static uint8_t encode(int v, int mn, int s) {
    return (uint8_t)clampi(lqo_round_half_away((double)(v - mn) / s), 0, 15);
}

/* quant.cpp:64-104 */
int lqo_quantize_second_level(const int8_t* q, uint32_t n, uint32_t k, uint32_t g,
                              uint8_t* codes, uint8_t* scales, uint8_t* offsets) {
    if (n < 1 || k < 1) return fail("matrix dimensions must be >= 1");
    if (g < 1) return fail("group_size must be >= 1");
    if (k % g != 0) {
        snprintf(g_err, sizeof g_err, "k = %u not divisible by group_size = %u", k, g);
        return 1;
    }
    const uint32_t gpr = k / g;
    for (uint32_t i = 0; i < n; ++i) {
        for (uint32_t gi = 0; gi < gpr; ++gi) {
            const uint64_t base = (uint64_t)i * k + (uint64_t)gi * g;
            int mn = q[base], mx = q[base];
            for (uint32_t j = 1; j < g; ++j) {
                const int v = q[base + j];
                if (v < -119 || v > 119) {
                    snprintf(g_err, sizeof g_err,
                             "level-1 code %d outside [-119,119] at row %u", v, i);
                    return 1;
                }
                mn = v < mn ? v : mn;
                mx = v > mx ? v : mx;
            }
            if (q[base] < -119 || q[base] > 119) {
                snprintf(g_err, sizeof g_err, "level-1 code outside [-119,119] at row %u", i);
                return 1;
            }
            uint8_t s, a;
            group_params(mn, mx, &s, &a);
            scales[(uint64_t)i * gpr + gi] = s;
            offsets[(uint64_t)i * gpr + gi] = a;
            for (uint32_t j = 0; j < g; ++j) codes[base + j] = encode(q[base + j], mn, s);
        }
    }
    return 0;
}

/* quant.cpp:222-228 */
void lqo_pack_plain(const uint8_t* codes, uint64_t count, uint8_t* packed) {
    memset(packed, 0, (count + 1) / 2);
    for (uint64_t i = 0; i < count; ++i) {
        if (i % 2 == 0)
            packed[i / 2] |= codes[i] & 0x0F;
        else
            packed[i / 2] |= (uint8_t)(codes[i] << 4);
    }
}

/* quant.cpp:203-232 with layout = PlainRowMajor */
int lqo_build_bundle_plain(const float* w, uint32_t n, uint32_t k, uint32_t g,
                           uint8_t* packed, uint8_t* scales, uint8_t* offsets, float* cs) {
    const uint64_t nk = (uint64_t)n * k;
    int8_t* q = (int8_t*)malloc(nk ? nk : 1);
    uint8_t* codes = (uint8_t*)malloc(nk ? nk : 1);
    int rc = lqo_quantize_first_level(w, n, k, q, cs);
    if (!rc) rc = lqo_quantize_second_level(q, n, k, g, codes, scales, offsets);
    if (!rc) lqo_pack_plain(codes, nk, packed);
    free(q);
    free(codes);
    return rc;
}

/* packed.cpp:12-19 */
uint32_t lqo_pack_interleaved(const uint8_t* e) {
    uint32_t v = 0;
    for (int j = 0; j < 4; ++j) {
        const uint32_t byte = (e[j] & 0x0Fu) | ((e[j + 4] & 0x0Fu) << 4);
        v |= byte << (8 * j);
    }
    return v;
}

/* Dual-MMA record geometry with the default FragmentDescriptor
 * {warps 4, threads 32, mma_m 64, mma_k 32, 16 elems/thread/mma, dual span 64}
 * (layout.hpp:33-40). fragment_coords, layout.cpp:24-37:
 *   row = 16*warp + 8*r + thread/4
 *   col = 32*mma + 16*b + 4*(thread%4) + j
 * Record words: [even slab r0, even r1, odd r0, odd r1] (layout.cpp:56-72). */
static void dual_word_coords(uint32_t p, uint32_t w, uint32_t t, uint32_t half, uint32_t r,
                             uint32_t e, uint32_t* row, uint32_t* col) {
    const uint32_t b = e / 4, j = e % 4;
    *row = 16 * w + 8 * r + t / 4;
    *col = 32 * (2 * p + half) + 16 * b + 4 * (t % 4) + j;
}

/* layout.cpp:39-75 per 64-row band, bands in row order (bundle.cpp:251-274) */
int lqo_pack_dual(const uint8_t* codes, uint32_t n, uint32_t k, uint8_t* packed) {
    if (n % 64 != 0) return fail("dual-MMA layout needs n divisible by 64");
    if (k % 64 != 0) return fail("tile depth is not a multiple of dual_k_span");
    uint64_t off = 0;
    for (uint32_t band = 0; band < n / 64; ++band) {
        const uint8_t* bc = codes + (uint64_t)band * 64 * k;
        for (uint32_t p = 0; p < k / 64; ++p)
            for (uint32_t w = 0; w < 4; ++w)
                for (uint32_t t = 0; t < 32; ++t)
                    for (uint32_t half = 0; half < 2; ++half)
                        for (uint32_t r = 0; r < 2; ++r) {
                            uint8_t el[8];
                            for (uint32_t e = 0; e < 8; ++e) {
                                uint32_t row, col;
                                dual_word_coords(p, w, t, half, r, e, &row, &col);
                                el[e] = bc[(uint64_t)row * k + col];
                            }
                            const uint32_t word = lqo_pack_interleaved(el);
                            for (int bb = 0; bb < 4; ++bb)
                                packed[off++] = (uint8_t)(word >> (8 * bb));
                        }
    }
    return 0;
}

/* bundle.cpp:227-249 (+ unpack_dual_mma layout.cpp:77-112) */
int lqo_logical_codes(uint32_t n, uint32_t k, int layout, const uint8_t* packed,
                      uint8_t* codes) {
    const uint64_t nk = (uint64_t)n * k;
    if (layout == 0) {
        for (uint64_t i = 0; i < nk; ++i) {
            const uint8_t byte = packed[i / 2];
            codes[i] = (i % 2 == 0) ? (byte & 0x0F) : (byte >> 4);
        }
        return 0;
    }
    if (n % 64 != 0 || k % 64 != 0) return fail("dual-MMA layout needs n, k divisible by 64");
    uint64_t off = 0;
    for (uint32_t band = 0; band < n / 64; ++band) {
        uint8_t* bc = codes + (uint64_t)band * 64 * k;
        for (uint32_t p = 0; p < k / 64; ++p)
            for (uint32_t w = 0; w < 4; ++w)
                for (uint32_t t = 0; t < 32; ++t)
                    for (uint32_t half = 0; half < 2; ++half)
                        for (uint32_t r = 0; r < 2; ++r) {
                            const uint32_t word = (uint32_t)packed[off] |
                                                  (uint32_t)packed[off + 1] << 8 |
                                                  (uint32_t)packed[off + 2] << 16 |
                                                  (uint32_t)packed[off + 3] << 24;
                            off += 4;
                            const uint32_t lo = word & 0x0F0F0F0Fu, hi = (word >> 4) & 0x0F0F0F0Fu;
                            for (uint32_t e = 0; e < 8; ++e) {
                                uint32_t row, col;
                                dual_word_coords(p, w, t, half, r, e, &row, &col);
                                bc[(uint64_t)row * k + col] =
                                    (uint8_t)((e < 4 ? lo >> (8 * e) : hi >> (8 * (e - 4))) & 0xFF);
                            }
                        }
    }
    return 0;
}

/* bundle.cpp:89-135 */
int lqo_validate_bundle(uint32_t n, uint32_t k, uint32_t g, int layout, uint64_t packed_len,
                        const uint8_t* scales, const uint8_t* offsets, uint64_t ngroups,
                        const float* cs, uint32_t ncs) {
    if (n < 1 || k < 1) return fail("bundle dimensions must be >= 1");
    if (g < 1) return fail("group_size must be >= 1");
    if (k % g != 0) {
        snprintf(g_err, sizeof g_err, "k = %u not divisible by group_size = %u", k, g);
        return 1;
    }
    if (layout == 1) {
        if (n % 64 != 0) return fail("dual-MMA layout needs n divisible by 64");
        if (k % 64 != 0) return fail("dual-MMA layout needs k divisible by 64");
        if (g % 64 != 0)
            return fail("dual-MMA layout needs group_size divisible by 64 so each record word "
                        "pair stays within one group");
    }
    const uint64_t nk = (uint64_t)n * k;
    if (packed_len != (nk + 1) / 2) return fail("packed weight payload has wrong size");
    const uint32_t gpr = k / g;
    const uint64_t ng = (uint64_t)n * gpr;
    if (ngroups != ng) return fail("group parameter arrays have wrong size");
    if (ncs != n) return fail("channel scale array has wrong size");
    for (uint64_t i = 0; i < ng; ++i) {
        if (scales[i] < 1 || scales[i] > 16) {
            snprintf(g_err, sizeof g_err, "group scale %d out of [1,16] at row %u group %u",
                     scales[i], (uint32_t)(i / gpr), (uint32_t)(i % gpr));
            return 1;
        }
        if (offsets[i] < 9 || offsets[i] > 247) {
            snprintf(g_err, sizeof g_err, "group offset %d out of [9,247] at row %u group %u",
                     offsets[i], (uint32_t)(i / gpr), (uint32_t)(i % gpr));
            return 1;
        }
    }
    for (uint32_t r = 0; r < n; ++r) {
        const float s = cs[r];
        if (!(s > 0.0f) || !isfinite(s)) {
            snprintf(g_err, sizeof g_err, "channel scale at row %u must be positive and finite",
                     r);
            return 1;
        }
    }
    return 0;
}

/* quant.cpp:106-109 */
int8_t lqo_dequantize_scalar(uint8_t code, uint8_t s, uint8_t a) {
    const int group_min = (int)a - 128;
    return (int8_t)(int)(code * s + group_min);
}

/* quant.cpp:111-119 (Release mode) */
uint8_t lqo_dequantize_lane(uint8_t code, uint8_t s, uint8_t a) {
    const uint8_t biased = (uint8_t)((uint8_t)(code * s) + a);
    return (uint8_t)(biased ^ 0x80u);
}

/* packed.cpp:30-71: 2 AND + 1 SHR + 2 IMAD + 2 XOR */
int lqo_dequant_word(uint32_t w, uint8_t s, uint8_t a, uint32_t* lo, uint32_t* hi) {
    const uint32_t l = w & 0x0F0F0F0Fu;
    const uint32_t h = (w >> 4) & 0x0F0F0F0Fu;
    const uint32_t a4 = (uint32_t)a * 0x01010101u;
    *lo = (l * (uint32_t)s + a4) ^ 0x80808080u;
    *hi = (h * (uint32_t)s + a4) ^ 0x80808080u;
    return 7;
}

/* quant.cpp:234-251 */
int lqo_reconstruct_int8(uint32_t n, uint32_t k, uint32_t g, const uint8_t* codes,
                         const uint8_t* scales, const uint8_t* offsets, int8_t* out) {
    if (g < 1 || k % g != 0) return fail("k not divisible by group_size");
    const uint32_t gpr = k / g;
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t gi = 0; gi < gpr; ++gi) {
            const uint8_t s = scales[(uint64_t)i * gpr + gi], a = offsets[(uint64_t)i * gpr + gi];
            const uint64_t base = (uint64_t)i * k + (uint64_t)gi * g;
            for (uint32_t j = 0; j < g; ++j) out[base + j] = lqo_dequantize_scalar(codes[base + j], s, a);
        }
    return 0;
}

/* gemm.cpp:19-47 */
int lqo_quantize_activations(const float* x, uint32_t m, uint32_t k, int8_t* q, float* ts) {
    if (m < 1 || k < 1) return fail("activation dimensions must be >= 1");
    for (uint32_t i = 0; i < m; ++i) {
        const float* row = x + (uint64_t)i * k;
        float amax = 0.0f;
        for (uint32_t l = 0; l < k; ++l) {
            if (!isfinite(row[l])) {
                snprintf(g_err, sizeof g_err, "non-finite activation at (%u, %u)", i, l);
                return 1;
            }
            const float a = fabsf(row[l]);
            amax = amax < a ? a : amax;
        }
        const float s = amax == 0.0f ? 1.0f : amax / 127.0f;
        ts[i] = s;
        for (uint32_t l = 0; l < k; ++l)
            q[(uint64_t)i * k + l] =
                (int8_t)clampi(lqo_round_half_away((double)row[l] / s), -127, 127);
    }
    return 0;
}

/* quant.cpp:125-127 */
float lqo_epilogue(int64_t acc, float cs, float ts) {
    return (float)((double)acc * (double)cs * (double)ts);
}

/* gemm.cpp:53-57 */
int lqo_check_accumulator_range(uint32_t k) {
    return (int64_t)k * 127 * 127 >= ((int64_t)1 << 31) ? 1 : 0;
}

/* gemm.cpp:225-243 */
int lqo_gemm_oracle(const int8_t* q, const float* ts, uint32_t m, uint32_t k, const int8_t* w,
                    const float* cs, uint32_t n, int64_t* acc, float* y) {
    for (uint32_t i = 0; i < m; ++i) {
        const int8_t* xr = q + (uint64_t)i * k;
        for (uint32_t j = 0; j < n; ++j) {
            const int8_t* wr = w + (uint64_t)j * k;
            int64_t s = 0;
            for (uint32_t l = 0; l < k; ++l) s += (int64_t)xr[l] * (int64_t)wr[l];
            if (acc) acc[(uint64_t)i * n + j] = s;
            if (y) y[(uint64_t)i * n + j] = lqo_epilogue(s, cs[j], ts[i]);
        }
    }
    return 0;
}
