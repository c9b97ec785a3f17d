/* lqg — B200-native (sm_100a) LiquidGEMM W4A8 GEMM behind a plain C ABI.
 *
 * Drop-in boundary for the reference's W4A8 path (namespace lq,
 * /root/reference/proj):
 *
 *   lq::gemm_w4a8_accum(const ActivationQuant&, const QuantizedWeightBundle&,
 *                       const TileConfig&, Engine)        include/lq/gemm.hpp:49-51
 *   lq::gemm_w4a8(...same...)                             include/lq/gemm.hpp:54-55
 *
 * The reference passes host std::vectors and returns by value; this ABI splits
 * that into (1) a one-off weight upload + prepack (lqg_weights_create, the
 * analogue of to_dual_mma / pack_dual_mma, bundle.cpp:251-274), (2) async
 * device-pointer GEMM launches on a caller stream, and (3) a synchronous
 * host-buffer call with the reference's exact calling convention
 * (lqg_gemm_w4a8_host), which is what INTEGRATION.md binds lq::gemm_w4a8 to.
 *
 * No torch types, no C++ types: plain pointers and sizes. Streams are passed
 * as void* (a cudaStream_t / CUstream; NULL = legacy default stream).
 *
 * Status codes mirror the reference error taxonomy (errors.hpp:15-28 and the
 * CLI exit codes, cli.cpp:392-404):
 *   LQG_OK 0, LQG_EVALIDATION 1 (lq::ValidationError),
 *   LQG_EVERIFICATION 2 (lq::VerificationError), LQG_EIO 3 (lq::IoError),
 *   LQG_ECUDA 4, LQG_ENCCL 5, LQG_EUNSUPPORTED 6 (needs an sm_100 device).
 * The message of the last failure on the calling thread is lqg_last_error().
 *
 * There is no CPU fallback: every compute entry point runs the sm_100a
 * kernels in liblqg.so or fails with LQG_ECUDA / LQG_EUNSUPPORTED.
 */
#ifndef LQG_H
#define LQG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    LQG_OK = 0,
    LQG_EVALIDATION = 1,
    LQG_EVERIFICATION = 2,
    LQG_EIO = 3,
    LQG_ECUDA = 4,
    LQG_ENCCL = 5,
    LQG_EUNSUPPORTED = 6
};

/* Output element types for lqg_gemm_w4a8 / lqg_gemm_w4a8_host. F32 is
 * bit-identical to the reference's float output (quant.cpp:125-127 evaluated
 * in double, one rounding); F16/BF16 are round-to-nearest-even of that F32. */
enum { LQG_Y_F32 = 0, LQG_Y_F16 = 1, LQG_Y_BF16 = 2 };

/* Weight layouts of the reference bundle (bundle.hpp:36-39). */
enum { LQG_LAYOUT_PLAIN = 0, LQG_LAYOUT_DUAL_MMA = 1 };

/* Host view of an lq::QuantizedWeightBundle (bundle.hpp:41-69). The arrays
 * are borrowed for the duration of lqg_weights_create only.
 *   packed_weights: (n*k+1)/2 bytes, plain (element 2j in the low nibble of
 *                   byte j, quant.cpp:222-228) or dual-MMA records
 *                   (layout.hpp:1-23, FragmentDescriptor below).
 *   group_scales, group_offsets: n*(k/group_size) bytes, index r*(k/g)+g.
 *   channel_scales: n floats. */
typedef struct lqg_fragment_descriptor {
    uint8_t warps_per_group;              /* 4  (layout.hpp:34) */
    uint8_t threads_per_warp;             /* 32 */
    uint16_t mma_m;                       /* 64 */
    uint16_t mma_k;                       /* 32 */
    uint16_t elements_per_thread_per_mma; /* 16 */
    uint16_t dual_k_span;                 /* 64 */
} lqg_fragment_descriptor;

typedef struct lqg_bundle_view {
    uint32_t n, k, group_size;
    uint32_t layout; /* LQG_LAYOUT_* */
    lqg_fragment_descriptor fragment; /* meaningful for LQG_LAYOUT_DUAL_MMA */
    const uint8_t* packed_weights;
    uint64_t packed_bytes;
    const uint8_t* group_scales;
    const uint8_t* group_offsets;
    uint64_t n_groups;
    const float* channel_scales;
} lqg_bundle_view;

typedef struct lqg_weights lqg_weights; /* opaque, device-resident, immutable */

/* Host-only check with the reference's rules and messages
 * (QuantizedWeightBundle::validate, bundle.cpp:89-135, and
 * FragmentDescriptor::validate, layout.cpp:10-22). No GPU needed.
 * lqg_weights_create additionally rejects (LQG_EVALIDATION) what the device
 * layout cannot represent: group_size % 32 != 0. */
int lqg_bundle_validate(const lqg_bundle_view* bundle);

/* Validates exactly like QuantizedWeightBundle::validate (bundle.cpp:89-135),
 * prepacks into the device layout and uploads to
 * `device`. Synchronous. Replaces the reference's per-call layout work
 * (gemm.cpp:151-165). */
int lqg_weights_create(const lqg_bundle_view* bundle, int device, lqg_weights** out);

/* Device image (prepacked layout) size in bytes for an
 * n x k bundle with this group size; 0 if the device layout cannot hold it. */
uint64_t lqg_image_bytes(uint32_t n, uint32_t k, uint32_t group_size);

/* Host-only prepack (no GPU needed): validates like lqg_weights_create and
 * writes the device image into `image` (lqg_image_bytes bytes). Lets callers
 * prepack once offline and cache the result (see lqg_weights_from_image). */
int lqg_prepack_host(const lqg_bundle_view* bundle, uint8_t* image, uint64_t image_bytes);

/* Uploads a prepacked image (from lqg_prepack_host or a cache file) plus the n
 * channel scales to `device`. */
int lqg_weights_from_image(const uint8_t* image, uint64_t image_bytes, const float* channel_scales,
                           uint32_t n, uint32_t k, uint32_t group_size, int device,
                           lqg_weights** out);

/* Quantizes device FP32 weights w[n][k] (row pitch ldw floats) on the GPU with
 * the reference's two-level LiquidQuant quantizer (build_bundle,
 * quant.cpp:203-232; bit-exact) straight into the device layout. */
int lqg_weights_quantize(const float* d_w, int64_t ldw, uint32_t n, uint32_t k,
                         uint32_t group_size, void* stream, lqg_weights** out);

/* LQWB bundle files: the reference's on-disk format (bundle.hpp:5-24,
 * save_bundle / load_bundle, bundle.cpp:137-224), little-endian.
 * lqg_weights_load = load_bundle + lqg_weights_create: the reference's
 * read_bundle checks in its order and with its messages (bad magic, version,
 * layout flag, dimensions, truncation as LQG_EIO "... (byte offset N)",
 * trailing bytes) and then QuantizedWeightBundle::validate; plain-layout
 * payloads are prepacked on the device.
 * lqg_bundle_file_validate: the same checks, host only (no GPU).
 * lqg_weights_save: the handle as a PlainRowMajor LQWB file that the
 * reference's load_bundle reads back. */
int lqg_weights_load(const char* path, int device, lqg_weights** out);
int lqg_bundle_file_validate(const char* path);
int lqg_weights_save(const lqg_weights* w, const char* path);

int lqg_weights_destroy(lqg_weights* w);

/* n, k, group_size of the handle. */
int lqg_weights_shape(const lqg_weights* w, uint32_t* n, uint32_t* k, uint32_t* group_size);

/* Copies the handle back out as a plain-layout host bundle (the caller
 * provides packed (n*k+1)/2 bytes, n*(k/g) scales and offsets, n floats). */
int lqg_weights_export(const lqg_weights* w, uint8_t* packed, uint8_t* group_scales,
                       uint8_t* group_offsets, float* channel_scales);

/* Device bytes the handle streams per GEMM (prepacked codes + group params +
 * channel scales): the weight term of the roofline. */
uint64_t lqg_weights_device_bytes(const lqg_weights* w);

/* Split-K workspace (~23.6 MB of device memory). Passing ws = NULL uses the
 * default workspace of the (device, stream) pair: shared by every handle,
 * created on the first launch on that stream (one synchronous
 * initialisation, legal during CUDA-graph capture) and kept for the life of
 * the process. Launches on one stream are ordered, so they may share it;
 * launches on different streams get different ones. A graph captured on a
 * stream uses that stream's workspace: do not replay it concurrently with
 * other launches captured on or issued to the same stream without passing an
 * explicit workspace. Workspaces are initialised on creation and left in
 * that state by every launch. */
typedef struct lqg_workspace lqg_workspace;
int lqg_workspace_create(int device, lqg_workspace** out);
int lqg_workspace_destroy(lqg_workspace* ws);

/* Y[m][n] = (sum_k X[m][k] * W^[n][k]) * channel_scale[n] * token_scale[m]
 * (gemm.cpp:213-223), all device pointers, async on `stream`.
 *   d_x: m rows of int8 codes, row pitch ldx bytes (ldx % 16 == 0, ldx >= k).
 *   d_token_scales: m floats.
 *   d_y: m rows, row pitch ldy elements of y_dtype.
 *   ws: NULL = the default workspace of (device, stream), see above.
 * Rejects (LQG_EVALIDATION) m < 1 and k*127*127 >= 2^31 (gemm.cpp:53-57). */
int lqg_gemm_w4a8(const lqg_weights* w, const int8_t* d_x, int64_t ldx,
                  const float* d_token_scales, uint32_t m, void* d_y, int64_t ldy, int y_dtype,
                  lqg_workspace* ws, void* stream);

/* lqg_gemm_w4a8 whose epilogue stores every output tile into n_ys (1..8)
 * destinations with the same pitch: d_ys[0] plus up to 7 more, typically
 * the peers' Y buffers mapped over NVLink (CUDA IPC / symmetric memory). In
 * the N-split driver each rank passes its column slice of every rank's full
 * Y (base + column offset, ldy = n_full), so the row-output all-gather
 * happens inside the GEMM epilogue, tile by tile, overlapped with the
 * mainloop; the caller then only needs a cross-GPU barrier. Values are
 * bit-identical to lqg_gemm_w4a8. */
int lqg_gemm_w4a8_fanout(const lqg_weights* w, const int8_t* d_x, int64_t ldx,
                         const float* d_token_scales, uint32_t m, void* const* d_ys,
                         uint32_t n_ys, int64_t ldy, int y_dtype, lqg_workspace* ws,
                         void* stream);

/* INT32 accumulators only (gemm.cpp:138-211), bit-exact. d_acc: m x ldacc. */
int lqg_gemm_w4a8_accum(const lqg_weights* w, const int8_t* d_x, int64_t ldx, uint32_t m,
                        int32_t* d_acc, int64_t ldacc, lqg_workspace* ws, void* stream);

/* Grouped (MoE) W4A8 GEMM: num_groups problems that share n, k and group size
 * (the experts of one layer, BASELINE config 5 / the paper's MoE case, P:615,
 * P:618) in ONE persistent launch -- stream-K over the union of all groups'
 * tiles, so small experts do not each pay a launch and a tail. Group e owns
 * the m[e] rows starting at row0_e = m[0] + ... + m[e-1] of d_x (int8 codes,
 * pitch ldx), d_token_scales and d_y (pitch ldy): the expert-sorted token
 * layout. m[e] may be 0. weights[e] are handles on the same device.
 * Per group the result is bit-identical to lqg_gemm_w4a8 on that group alone
 * (and hence to the reference's gemm_w4a8, gemm.cpp:213-223).
 * 1 <= num_groups <= 64. */
int lqg_gemm_w4a8_grouped(const lqg_weights* const* weights, uint32_t num_groups,
                          const int8_t* d_x, int64_t ldx, const float* d_token_scales,
                          const uint32_t* m, void* d_y, int64_t ldy, int y_dtype,
                          lqg_workspace* ws, void* stream);
/* INT32 accumulators of the grouped GEMM (gemm.cpp:138-211 per group). */
int lqg_gemm_w4a8_grouped_accum(const lqg_weights* const* weights, uint32_t num_groups,
                                const int8_t* d_x, int64_t ldx, const uint32_t* m,
                                int32_t* d_acc, int64_t ldacc, lqg_workspace* ws, void* stream);

/* Host-buffer call with the reference's convention: x is m*k int8 codes
 * (row-major, ActivationQuant::values, gemm.hpp:35-39), token_scales m floats,
 * y receives m*n values of y_dtype, row-major. Stages through device buffers
 * taken from a process-wide pool (one staging context per concurrent call)
 * on `stream` and returns after y is written (like the reference, which
 * returns by value). Re-entrant: any number of host threads may call it on
 * the same or different handles (the handle is never modified). */
int lqg_gemm_w4a8_host(const lqg_weights* w, const int8_t* x, const float* token_scales,
                       uint32_t m, void* y, int y_dtype, void* stream);
int lqg_gemm_w4a8_accum_host(const lqg_weights* w, const int8_t* x, uint32_t m, int32_t* acc,
                             void* stream);

/* The dequantized INT8 weights W^[n][k] (reconstruct_int8, quant.cpp:234-251),
 * produced by the same device dequant code the GEMM mainloop runs. d_w: n x ldw. */
int lqg_dequant_weights(const lqg_weights* w, int8_t* d_w, int64_t ldw, void* stream);

/* Per-token activation quantization on the GPU (gemm.cpp:19-47, bit-exact):
 * d_x m x k floats (pitch ldx floats) -> d_q m x k int8 (pitch ldq bytes),
 * d_ts m floats. Non-finite inputs -> LQG_EVALIDATION after the stream sync
 * that this call performs only when check_finite != 0. */
int lqg_quantize_activations(const float* d_x, int64_t ldx, uint32_t m, uint32_t k,
                             int8_t* d_q, int64_t ldq, float* d_ts, int check_finite,
                             void* stream);

/* Number of kernels liblqg.so launched on this process so far (all entry
 * points). The bench reports the delta over its timed region. */
uint64_t lqg_kernel_launch_count(void);

/* Launch-schedule knobs (tuning and testing hook, process-wide): token-tile
 * cap "max_bn", CTA pairs "pair" (-1 auto, 0 never, 1 wherever legal),
 * "pair_min_m", "pair_single_tile", ring split "x_ring_bytes",
 * "max_x_stages", "max_w_stages" (ring depths are rounded down to even),
 * "grid", "raster_gm", "no_dp", "no_pdl", "acc_stages" (1: one accumulator
 * stage and a deeper TMEM A ring), "no_quad" (1: split tiles exchange
 * partials through L2 even where 4-CTA clusters fit), "auto_tile" (0: skip
 * the short-k / few-tile / small-weight token-tile and pair corrections;
 * they apply only while "max_bn" and "pair" keep their defaults), and for the host-buffer
 * calls "host_chunk_m", "host_chunks" (row-chunk pipelining).
 * Results are bit-identical under every setting; only the schedule changes.
 * Unknown names and out-of-range values -> LQG_EVALIDATION. */
int lqg_tune_set(const char* name, int64_t value);
int lqg_tune_get(const char* name, int64_t* value);
void lqg_tune_reset(void);

const char* lqg_last_error(void);
const char* lqg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LQG_H */
