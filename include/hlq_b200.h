/*
 * hlq_b200.h -- C ABI of the B200 (sm_100a) HLQ backward path.
 *
 * This is the drop-in boundary for the reference's HLQ hot path
 * (/root/reference/pkg/src/hlq).  The reference is a pure-Python/numpy package
 * with no FFI; its interface for this path is a set of Python functions.  Each
 * entry point below replaces one of them (file:line cited per function) and is
 * what a ctypes / cffi binding of that function would call -- see
 * INTEGRATION.md for the binding a maintainer would add.
 *
 * Conventions
 *  - every pointer is a DEVICE pointer unless stated otherwise; the caller
 *    allocates every output and workspace (the library never allocates device
 *    memory, so every call is CUDA-graph-capture safe);
 *  - all work is enqueued on `stream` (a cudaStream_t passed as void*);
 *  - shapes / strides are int64_t element counts, row-major;
 *  - return value is an hlq_status; hlq_last_error() gives a message
 *    (thread-local).  Status codes map onto the reference's exception classes
 *    (errors.py:4-13): DIMENSION -> DimensionError, PARAMETER -> ParameterError,
 *    STATE -> StateError, NONFINITE -> ValueError.
 *  - "codes" are int8 quantizer outputs; operand layouts are K-major (each row
 *    holds one output row/column's contraction axis), which is the layout
 *    tcgen05 consumes directly.
 *  - block size is 16 (hadamard.py:19, the HLQ design point); `bitmap` has bit
 *    i set iff Walsh basis i is kept (hadamard.py:97-106).
 */
#ifndef HLQ_B200_H
#define HLQ_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HLQ_API __attribute__((visibility("default")))
#else
#define HLQ_API
#endif

/* Device scratch the single-call quantizers need for their statistics, the
 * fused kernel's grid barrier and its work-ticket counters, each on its own
 * 128-byte line (zeroed by the library on the caller's stream).  The
 * single-call quantizers (hlq_quantize_ht_cols / _proj_rows / _dual* and
 * hlq_conv_acbp_compress) also accept stats_ws = NULL: the statistics then
 * live in one of 64 library-owned per-device slots that the fused launch
 * zeroes again when it finishes (no memset launch; fewer than 64 such calls
 * may execute concurrently on a device), and are not returned. */
#define HLQ_STATS_WS_BYTES 512

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HLQ_OK = 0,
  HLQ_ERR_DIMENSION = 1, /* errors.py:4  DimensionError */
  HLQ_ERR_PARAMETER = 2, /* errors.py:8  ParameterError */
  HLQ_ERR_STATE = 3,     /* errors.py:12 StateError */
  HLQ_ERR_NONFINITE = 4, /* quantize.py:138-139 ValueError */
  HLQ_ERR_CUDA = 5,
  HLQ_ERR_FORMAT = 6 /* malformed ACBP container: FormatError; hlq_last_error_offset() = byte offset */
} hlq_status;

typedef enum { HLQ_F32 = 0, HLQ_BF16 = 1 } hlq_dtype;

typedef enum {
  HLQ_EPI_EXACT = 0, /* out = f32(f64(acc) * (f64(f32(sa*sb)) * extra)), quantize.py:181-187 */
  HLQ_EPI_FAST = 1   /* out = f32(acc) * f32(sa*sb*extra); training path, fp32 or bf16 out */
} hlq_epilogue;

/* Library identification. */
HLQ_API const char* hlq_version(void);
/* Message of the last failing call on this thread ("" if none). */
HLQ_API const char* hlq_last_error(void);
/* 1 when a sm_100 device and the driver entry points are usable, else 0. */
HLQ_API int hlq_device_ok(void);

/* ---------------------------------------------------------------------------
 * Stage primitives
 * ------------------------------------------------------------------------- */

/* Q_bits( block-FWHT along the contiguous axis of src (rows x cols) ).
 * Replaces `_block_axis(gy, 2, plan)` + `quant_pseudo_stochastic` on the gx
 * left operand (backprop.py:212-220,362,367; quantize.py:128-145).
 * Writes codes (rows x pad16(cols), leading dim ld_dst >= pad16(cols), a
 * multiple of 16) and the fp32 scale.  stats_ws: HLQ_STATS_WS_BYTES device
 * scratch; on return stats_ws[0] holds the bits of max|4v| (>= 0x7F800000
 * means a NaN/Inf was present, the reference's ValueError).  bits in {4, 8}. */
HLQ_API int hlq_quantize_ht_cols(const void* src, int dtype, int64_t rows, int64_t cols, int64_t ld_src,
                         int bits, uint32_t* stats_ws, int8_t* dst, int64_t ld_dst,
                         float* scale_out, void* stream);

/* Q_bits( rank-r block projection along the ROW axis of src ), codes written
 * transposed: dst[c * ld_dst + (s * nblk + blk) * r + j], nblk = ceil(rows/16).
 * src is `segs` segments of (rows x cols) with row stride ld_src and segment
 * stride seg_src.  Replaces `_project_axis` + `quant_pseudo_stochastic`
 * (backprop.py:223-234; acbp_compress :373-385; hlq_grad_weight :401-407) and,
 * with bitmap 0xFFFF, `_block_axis(w, 0, plan)` (:363).  stats_ws: HLQ_STATS_WS_BYTES of
 * scratch, the amax bits land in stats_ws[2]. */
HLQ_API int hlq_quantize_proj_rows(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                           int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits,
                           uint32_t* stats_ws, int8_t* dst, int64_t ld_dst, float* scale_out,
                           void* stream);

/* Both gy operands in ONE read of gy per pass (the fused "dual" transform):
 * the gx codes Q_bits_gx(HT along cols) exactly as hlq_quantize_ht_cols and
 * the gw codes Q_bits_gw(projection along rows) exactly as
 * hlq_quantize_proj_rows, over the same (segs x rows x cols) view.  Valid when
 * the token axis is the projection axis (reference axis rule L >= 16, or
 * L == 1 with projection along the batch).  stats_ws: HLQ_STATS_WS_BYTES. */
HLQ_API int hlq_quantize_dual(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                              int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits_gx,
                              int bits_gw, uint32_t* stats_ws, int8_t* dst_gx, int64_t ld_gx,
                              int8_t* dst_gw, int64_t ld_gw, float* scale_gx, float* scale_gw,
                              void* stream);

/* hlq_quantize_dual plus the fp32 column sums of the source (colsum_out, cols
 * floats): the bias gradient gy.sum over tokens (harness/layers.py:67 before
 * its /B), read from the same tiles as the STATS pass -- no separate pass
 * over gy.  Deterministic: per-work-item partials in colsum_ws
 * (hlq_quantize_dual_colsum_ws bytes), reduced in a fixed order inside the
 * same launch. */
HLQ_API size_t hlq_quantize_dual_colsum_ws(int64_t segs, int64_t rows, int64_t cols, uint32_t bitmap);
HLQ_API int hlq_quantize_dual_colsum(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                                     int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits_gx,
                                     int bits_gw, uint32_t* stats_ws, int8_t* dst_gx, int64_t ld_gx,
                                     int8_t* dst_gw, int64_t ld_gw, float* scale_gx, float* scale_gw,
                                     float* colsum_out, void* colsum_ws, size_t colsum_ws_bytes, void* stream);

/* hlq_quantize_dual_colsum with the gx codes optionally PACKED int4 (pack_gx = 1,
 * bits_gx = 4): two codes per byte, low nibble first (acbp.py:56-61), row
 * stride ld_gx bytes >= pad16(cols) / 2 (a multiple of 16) -- the A operand of
 * hlq_gemm_i4a_ex / hlq_gemm_desc.a_packed.  colsum_out may be NULL (no column
 * sums).  Same codes and scales as the int8 form. */
HLQ_API int hlq_quantize_dual_ex(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                                 int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits_gx, int bits_gw,
                                 uint32_t* stats_ws, void* dst_gx, int64_t ld_gx, int pack_gx, int8_t* dst_gw,
                                 int64_t ld_gw, float* scale_gx, float* scale_gw, float* colsum_out,
                                 void* colsum_ws, size_t colsum_ws_bytes, void* stream);

/* The two passes of hlq_quantize_proj_rows, separately, for the data-parallel
 * global-scale mode: _amax accumulates (atomic max, no reset) the transformed
 * statistics into stats[2..3] (stats: 4 x uint32, zero-initialised by the
 * caller); callers all-reduce(MAX) the 4 words across ranks, then _quant
 * quantizes with scale = amax / qmax (quantize.py:94-100). */
HLQ_API int hlq_proj_rows_amax(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                       int64_t ld_src, int64_t seg_src, uint32_t bitmap, uint32_t* stats,
                       void* stream);
HLQ_API int hlq_proj_rows_quant(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                        int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits,
                        const uint32_t* stats, int8_t* dst, int64_t ld_dst, float* scale_out,
                        void* stream);

/* One pass of the general transform (the building block of every call above):
 * mode 0 = STATS (max-accumulates {amax, ~minnz} of the gx operand into
 * stats[0..1] and of the gw operand into stats[2..3]; the caller zeroes
 * stats first, or all-reduces(MAX) them across ranks in between), mode 1 =
 * QUANT with the scales implied by `stats`.  This is what the exact
 * data-parallel mode uses: STATS on the local shard, all-reduce(MAX) of the 4
 * words, QUANT -- every rank then quantizes with the scale the single-process
 * reference computes. */
HLQ_API int hlq_transform_pass(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                               int64_t ld_src, int64_t seg_src, int do_gx, int do_gw,
                               uint32_t bitmap, int bits_gx, int bits_gw, int mode, uint32_t* stats,
                               int8_t* dst_gx, int64_t ld_gx, int8_t* dst_gw, int64_t ld_gw,
                               float* scale_gx, float* scale_gw, void* stream);

/* D[m, n] = sum_k A[m, k] * B[n, k] on int8 codes (tcgen05 kind::i8, int32 in
 * TMEM), dequantized with the fused epilogue.  Replaces `int_matmul` +
 * `int_matmul_dequant` (quantize.py:152-187).  lda/ldb are byte strides,
 * multiples of 16; sa/sb are device fp32 scales.  out may be NULL; acc_out
 * (int32, M x N, ld_acc) may be NULL -- it exposes the exact accumulator for
 * parity checks.  Fails with PARAMETER if K * qmax_a * qmax_b could overflow
 * int32 (pass the operands' bit widths). */
HLQ_API int hlq_gemm_i8(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int64_t M, int64_t N,
                int64_t K, int bits_a, int bits_b, const float* sa, const float* sb, double extra,
                int epilogue, void* out, int out_dtype, int64_t ldo, int32_t* acc_out,
                int64_t ld_acc, void* stream);

/* Grouped form: the contraction runs over `groups` stacked K panels,
 * D[m, n] = sum_g sum_k A[g][m, k] * B[g][n, k], panel g of A at byte offset
 * g * a_gstride (likewise B).  This is the batch-axis projection with L > 1,
 * whose reference K index is (block, basis, l) (backprop.py:223-234,402-403). */
HLQ_API int hlq_gemm_i8_grouped(const int8_t* A, int64_t lda, int64_t a_gstride, const int8_t* B,
                        int64_t ldb, int64_t b_gstride, int64_t M, int64_t N, int64_t K,
                        int64_t groups, int bits_a, int bits_b, const float* sa, const float* sb,
                        double extra, int epilogue, void* out, int out_dtype, int64_t ldo,
                        int32_t* acc_out, int64_t ld_acc, void* stream);

/* Split-K form of hlq_gemm_i8_grouped for products with few output tiles
 * and a long contraction (the dW GEMM: M = O, N = I, K = projected tokens).
 * ws (device, caller-allocated, no initialisation needed) of at least
 * hlq_gemm_i8_ws(M, N, K, groups) bytes lets the kernel split K across CTAs;
 * the per-split int32 partial tiles are summed in-kernel (exact) before the
 * same dequant epilogue.  ws == NULL or too small runs unsplit.  Same
 * contract and results as hlq_gemm_i8_grouped (int_matmul_dequant,
 * quantize.py:152-187). */
HLQ_API size_t hlq_gemm_i8_ws(int64_t M, int64_t N, int64_t K, int64_t groups);
/* Contractions longer than the int32-exact bound (K * groups * qmax_a * qmax_b
 * >= 2^31, e.g. an 8-bit dW with K > 133,143) run as K chunks that each stay
 * inside it, summed in int64 before the dequant -- the reference accumulates
 * in int64 up to MAX_K = {8: 10^6, 4: 10^7} (quantize.py:19-21,166-170) and
 * hlq_gemm_i8_ex fails with PARAMETER past that bound, as int_matmul does.
 * Such products need ws of hlq_gemm_i8_ws_bits(...) bytes (they cannot run
 * unsplit) and acc_out == NULL (an int32 dump could overflow). */
HLQ_API size_t hlq_gemm_i8_ws_bits(int64_t M, int64_t N, int64_t K, int64_t groups, int bits_a, int bits_b);
HLQ_API int hlq_gemm_i8_ex(const int8_t* A, int64_t lda, int64_t a_gstride, const int8_t* B,
                           int64_t ldb, int64_t b_gstride, int64_t M, int64_t N, int64_t K,
                           int64_t groups, int bits_a, int bits_b, const float* sa, const float* sb,
                           double extra, int epilogue, void* out, int out_dtype, int64_t ldo,
                           int32_t* acc_out, int64_t ld_acc, void* ws, size_t ws_bytes,
                           void* stream);

/* hlq_gemm_i8_ex with the A operand as PACKED int4 codes: two codes per byte,
 * low nibble first (the ACBP container's nibble order, acbp.py:56-61), i.e.
 * A[m, k] is the signed nibble (k & 1 ? high : low) of byte A[m * lda + k/2];
 * lda (bytes, a multiple of 16) >= ceil(K/2).  bits_a must be 4.  The GEMM
 * sign-extends the nibbles to int8 in shared memory ahead of the tcgen05
 * kind::i8 MMAs (sm_100a has no int4 MMA): half the A bytes of the int8 form,
 * same results bit for bit. */
HLQ_API int hlq_gemm_i4a_ex(const uint8_t* A, int64_t lda, int64_t a_gstride, const int8_t* B, int64_t ldb,
                            int64_t b_gstride, int64_t M, int64_t N, int64_t K, int64_t groups, int bits_b,
                            const float* sa, const float* sb, double extra, int epilogue, void* out,
                            int out_dtype, int64_t ldo, void* ws, size_t ws_bytes, void* stream);

/* One product for hlq_gemm_i8_multi (fields as in hlq_gemm_i8_grouped). */
typedef struct {
  const int8_t* A;
  int64_t lda, a_gstride;
  const int8_t* B;
  int64_t ldb, b_gstride;
  int64_t M, N, K, groups;
  int bits_a, bits_b;
  const float* sa;
  const float* sb;
  double extra;
  int epilogue;
  void* out;
  int out_dtype;
  int64_t ldo;
  int32_t* acc_out;
  int64_t ld_acc;
  int a_packed;  /* 1: A holds packed int4 codes (see hlq_gemm_i4a_ex); bits_a must be 4 */
} hlq_gemm_desc;

/* n (1 or 2) independent products -- typically a layer's dX and dW GEMMs --
 * with hlq_gemm_i8_grouped's contract each.  When both have long
 * contractions they run as ONE CTA-pair launch whose clusters take a
 * longest-first static schedule over both products' tiles (a layer's few long
 * dW tiles and many short dX tiles then pack evenly across the SMs instead of
 * running as two partially-filled waves); otherwise as separate launches. */
HLQ_API int hlq_gemm_i8_multi(int n, const hlq_gemm_desc* descs, void* stream);

/* ---------------------------------------------------------------------------
 * Reference-function equivalents (whole calls)
 * ------------------------------------------------------------------------- */

/* Payload geometry of acbp_compress for x of shape (B, L, I):
 *   axis 1 (tokens): I rows of K = B * ceil(L/16) * r codes;
 *   axis 0 (batch):  L*I rows (row l*I + i) of K = ceil(B/16) * r codes.
 * hlq_acbp_k returns K (per row), hlq_acbp_rows the row count. */
HLQ_API int64_t hlq_acbp_k(int64_t B, int64_t L, int axis, int rank);
HLQ_API int64_t hlq_acbp_rows(int64_t L, int64_t I, int axis);

/* backprop.py:373-385  acbp_compress(x, plan, bits, pad_small_axes).
 * x is (B, L, I); axis from ht_axis_for (0 = batch, 1 = tokens).  Payload is
 * written K-major, payload[row * ld_payload + k] (the reference's (K, I)
 * payload, transposed; see hlq_acbp_k).  stats_ws: HLQ_STATS_WS_BYTES of scratch. */
HLQ_API int hlq_acbp_compress(const void* x, int dtype, int64_t B, int64_t L, int64_t I, int axis,
                      uint32_t bitmap, int bits, int8_t* payload, int64_t ld_payload,
                      float* scale_out, uint32_t* stats_ws, void* stream);

/* Conv2d (harness/layers.py:96-158).  ACBP of the im2col'd input without
 * materialising it: x is channels-last (B, H, W, C); the payload row for
 * column (c, i, j) of cols is c*k*k + i*k + j (torch's weight flattening);
 * K = B * ceil(Ho*Wo/16) * rank.  Replaces Conv2d.forward's im2col +
 * acbp_compress (layers.py:141-151,46-55).  Requires Ho*Wo >= 16. */
HLQ_API int hlq_conv_acbp_compress(const void* x_nhwc, int dtype, int64_t B, int64_t H, int64_t W,
                                   int64_t C, int k, int stride, int pad, uint32_t bitmap,
                                   int bits, int8_t* payload, int64_t ld_payload, float* scale_out,
                                   uint32_t* stats_ws, void* stream);

/* One pass of hlq_conv_acbp_compress: mode 0 = STATS (max-accumulates into
 * stats_ws[2..3]; zero them first, or all-reduce(MAX) them across ranks
 * after), mode 1 = QUANT with the scale those statistics imply -- the exact
 * data-parallel mode's global-scale ACBP of a conv input (dp.ExactDP). */
HLQ_API int hlq_conv_acbp_pass(const void* x_nhwc, int dtype, int64_t B, int64_t H, int64_t W, int64_t C, int k,
                               int stride, int pad, uint32_t bitmap, int bits, int mode, uint32_t* stats_ws,
                               int8_t* payload, int64_t ld_payload, float* scale_out, void* stream);

/* True stochastic rounding (quantize.py:114-125), bit-exact with the
 * reference's RngState streams: codes of the transformed source with
 * up = f64(q - floor(q)) > U, U = the element's draw from numpy's
 * Philox4x64-10 keyed [seed, counter] (RngState(seed, counter).uniform over
 * the array the reference quantizes, C order).  seed = RngState.split(tag) of
 * the caller's state (tags backprop.py:42-43).  along_cols = 1: HT along cols
 * (the gx operand of gy; codes (segs*rows, ld_dst)); 0: projection along rows
 * keeping `bitmap` (gw operand / ACBP / W codes with bitmap 0xFFFF; codes
 * K-major per column, as hlq_quantize_proj_rows).  index_kind (rows mode):
 * 0 = the reference quantizes (cols, K) (gy's gw operand), 1 = (K, cols)
 * (ACBP payload, W), 2 = batch-axis gy with L > 1, cols = l2 * o2.
 * stats_ws: HLQ_STATS_WS_BYTES (the STATS pass runs inside). */
HLQ_API int hlq_quantize_stochastic(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                                    int64_t ld_src, int64_t seg_src, int along_cols, uint32_t bitmap,
                                    int bits, uint64_t seed, uint64_t counter, int index_kind, int64_t l2,
                                    int64_t o2, uint32_t* stats_ws, int8_t* dst, int64_t ld_dst,
                                    float* scale_out, void* stream);

/* Calibration energy (train.py:128-134 _basis_energy): energy16[i] = sum over
 * every 16-row block (zero-padded) and column of the source view of |c_i|, c
 * the orthonormal 16-point transform along rows -- the column sums of the
 * reference's per-block |coefficient| matrix, in fp64.  select_bases
 * (hadamard.py:174-188) keeps the `rank` largest means. */
HLQ_API int hlq_basis_energy(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                             int64_t ld_src, int64_t seg_src, double* energy16, void* stream);

/* ---- baseline strategies (backprop.py:91-155, 212-303) ----
 * A strided view of a float32 / bfloat16 source: unit (segment s, 16-block b
 * along rows, column c), element (s, r, c) at src + s*src_stride[0] +
 * r*src_stride[1] + c*src_stride[2].  bitmap selects the kept bases of the
 * orthonormal 16-point block transform along rows (0xFFFF: `_block_axis`,
 * backprop.py:212-220; a subset: `_project_axis`, :223-234); bitmap 0 is the
 * identity (no transform; r indexes the output).  Output element (s, k, c),
 * k = b*rank + j for the j-th kept basis (identity: k = r), is written at
 * dst + s*dst_stride[0] + k*dst_stride[1] + c*dst_stride[2]; idx_stride maps
 * it to its C-order index in the array the reference quantizes (the Philox
 * draw index of true stochastic rounding).  Rows past `rows` are zero padding
 * (transform) or absent (identity). */
typedef struct hlq_xform {
  const void* src;
  int32_t src_dtype;
  int64_t segs, rows, cols;
  int64_t src_stride[3];
  uint32_t bitmap;
  int64_t dst_stride[3];
  int64_t idx_stride[3];
} hlq_xform;

/* Q_bits of the view's outputs with ONE per-tensor scale (quantize.py:94-100):
 * rounding 0 = quant_pseudo_stochastic (quantize.py:128-145), 1 =
 * quant_stochastic with RngState(seed, counter) draws (quantize.py:114-125).
 * int8 codes at dst (positions the view does not write are left untouched:
 * zero them first when they are GEMM padding), scale_out one fp32, stats_ws
 * HLQ_STATS_WS_BYTES device bytes (word 0 = amax bits; >= 0x7F800000 flags a
 * non-finite input).  Two launches (statistics, quantization). */
HLQ_API int hlq_xform_quantize(const hlq_xform* view, int bits, int rounding, uint64_t seed, uint64_t counter,
                               uint32_t* stats_ws, int8_t* dst, float* scale_out, void* stream);

/* The view's outputs in float32 (the bits=None float pipelines and the
 * LBP-WHT low-rank projection, backprop.py:223-234). */
HLQ_API int hlq_xform_project_f32(const hlq_xform* view, float* dst, void* stream);

/* `_unproject_axis` (backprop.py:237-249): the view's SOURCE (float32) holds
 * kept coefficients (s, k, c); scatter them into full 16-blocks by bitmap,
 * inverse (= forward, orthonormal) transform, write rows r < rows as
 * (s, r, c) through dst_stride. */
HLQ_API int hlq_xform_unproject_f32(const hlq_xform* view, float* dst, void* stream);

/* The dX right operand of many layers at once: codes_i = Q_bits(HT_O(W_i))
 * for n <= 128 fp32 weights W_i (O_i x I_i, row-major), written K-major as
 * (I_i rows of ld_i >= pad16(O_i) bytes), scale_i one fp32 each -- identical
 * to hlq_quantize_proj_rows(W_i, 1, O_i, I_i, bitmap 0xFFFF) per tensor
 * (`_block_axis(w, 0, plan)` + `_quant`, backprop.py:363,368), in ONE
 * cooperative launch (training refreshes every layer's codes once per
 * optimizer step).  w, O, I, codes, ld, scales are HOST arrays of n entries
 * holding device pointers / extents.  ws: hlq_quantize_weights_ws(n) device
 * bytes (no initialisation needed). */
HLQ_API size_t hlq_quantize_weights_ws(int n);
HLQ_API int hlq_quantize_weights(int n, const float* const* w, const int64_t* O, const int64_t* I,
                                 int bits, int8_t* const* codes, const int64_t* ld,
                                 float* const* scales, uint32_t* ws, size_t ws_bytes, void* stream);
/* The same, also writing wbf16[i] (device, O_i x I_i row-major, may be a null
 * array) = RN-to-bf16 copy of W_i from the statistics pass's read: the forward
 * GEMM operand under bf16 autocast, without a separate cast per layer. */
HLQ_API int hlq_quantize_weights_ex(int n, const float* const* w, const int64_t* O, const int64_t* I,
                                    int bits, int8_t* const* codes, const int64_t* ld, float* const* scales,
                                    void* const* wbf16, uint32_t* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * ACBP container (acbp.py:3-212): the reference's bit-exact serialized form of
 * a compressed activation -- header, per-tensor scale, payload in the
 * reference's C order (int8, or int4 packed two per byte, low nibble first)
 * and a zlib CRC32 -- built and verified on the GPU.  Our payload is K-major
 * (rows = I, or L*I for the batch axis; K codes per row).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t B, L, I;            /* original activation shape */
  int bits, block, rank;
  uint32_t bitmap;
  int axis;                   /* the container's axis rule (acbp.py:_container_axis) */
  int64_t rows, K;            /* our K-major payload geometry */
  int64_t payload_bytes, total_bytes;
} hlq_acbp_info;

/* Container size: 33-byte header + scale, payload, 4-byte CRC. */
HLQ_API int64_t hlq_acbp_container_bytes(int64_t rows, int64_t k, int bits);
/* Device scratch for hlq_acbp_pack / hlq_acbp_unpack of a container of that size. */
HLQ_API size_t hlq_acbp_ws(int64_t total_bytes);
/* acbp_pack (acbp.py:76-96): out (device, exactly hlq_acbp_container_bytes
 * bytes) receives the container of the K-major payload (rows x k, ld), the
 * device fp32 scale and the plan / shape fields.  Stream-ordered. */
HLQ_API int hlq_acbp_pack(const int8_t* payload, int64_t ld, int64_t rows, int64_t k, int bits, int block,
                          uint32_t bitmap, int64_t B, int64_t L, int64_t I, const float* scale,
                          uint8_t* out, int64_t out_bytes, void* ws, size_t ws_bytes, void* stream);
/* acbp_unpack, header half (acbp.py:127-185): validates every header field and
 * the total length with the reference's rules; fills info.  Synchronous
 * (copies the 33 header bytes back).  HLQ_ERR_FORMAT + offset on violation. */
HLQ_API int hlq_acbp_parse(const uint8_t* buf, int64_t nbytes, hlq_acbp_info* info, void* stream);
/* acbp_unpack, payload half (acbp.py:186-207): range / padding / CRC checks in
 * the reference's order, then the payload back to K-major (rows x K, ld >= K)
 * and the scale.  Synchronous.  HLQ_ERR_FORMAT + offset on violation. */
HLQ_API int hlq_acbp_unpack(const uint8_t* buf, int64_t nbytes, const hlq_acbp_info* info, int8_t* payload,
                            int64_t ld, float* scale_out, void* ws, size_t ws_bytes, void* stream);
/* Byte offset of the last HLQ_ERR_FORMAT on this thread. */
HLQ_API int64_t hlq_last_error_offset(void);

/* Conv2d dX as ONE implicit GEMM (stride 1): dx[b, h, w, c] (channels-last)
 * = deq( sum over taps (i, j) and o of gcodes[b, h + pad - i, w + pad - j, o]
 *        * wcodes[c*k*k + i*k + j, o] ), zero outside the gy extent.  gcodes is
 * the gx operand of the conv backward (B, Ho, Wo, O) with pixel stride ld_g
 * (= hlq_quantize_dual's gx codes), wcodes the W codes (C*k*k rows of ld_w).
 * The taps accumulate in int32 before the dequant, so acc_out (B*H*W x C,
 * optional) equals col2im of the reference's per-tap int64 accumulators and dx
 * matches the reference's fp32 col2im (layers.py:109-121,153-158) to fp32
 * rounding rather than bit for bit.  Replaces GEMM -> dcols -> col2im. */
HLQ_API int hlq_conv_dgrad_i8(const int8_t* gcodes, int64_t ld_g, int64_t B, int64_t Ho, int64_t Wo,
                              int64_t O, const int8_t* wcodes, int64_t ld_w, int64_t C, int k,
                              int stride, int pad, int bits, const float* sg, const float* sw,
                              int epilogue, void* dx_nhwc, int dx_dtype, int32_t* acc_out,
                              void* stream);

/* Implicit-GEMM dgrad for any stride: dX (B, H, W, C) channels-last, H / W the
 * forward input extent ((H + 2 pad - k) / stride + 1 == Ho).  Stride s > 1 runs
 * as s^2 output phases (h = s h' + ph): phase (ph, pw) is a stride-1
 * correlation of the gy codes with the taps i = (ph + pad) mod s + s t -- no
 * zero-inserted gy, no dcols tensor -- and its rows are scattered to dX by the
 * epilogue (harness/layers.py:153-158 lowers this to GEMM + col2im).  Taps are
 * summed in int32 before the dequant, as at stride 1. */
HLQ_API int hlq_conv_dgrad_i8_ex(const int8_t* gcodes, int64_t ld_g, int64_t B, int64_t Ho, int64_t Wo, int64_t O,
                                 const int8_t* wcodes, int64_t ld_w, int64_t C, int k, int stride, int pad,
                                 int64_t H, int64_t W, int bits, const float* sg, const float* sw, int epilogue,
                                 void* dx_nhwc, int dx_dtype, int32_t* acc_out, void* stream);

/* col2im (layers.py:109-121): dx[b, h, w, c] (channels-last) = sum over taps
 * in the reference's (i, j) order of dcols[b*L + l, c*k*k + i*k + j]
 * (fp32 accumulation; bit-exact vs the reference for fp32 dcols). */
HLQ_API int hlq_col2im(const void* dcols, int dtype, int64_t ld, int64_t B, int64_t H, int64_t W,
                       int64_t C, int k, int stride, int pad, void* dx_nhwc, int out_dtype,
                       void* stream);

/* col2im with a choice of dcols column order: 0 = (c, tap) (= hlq_col2im),
 * 1 = (tap, c) -- what the dX GEMM produces when the W codes rows are
 * permuted tap-major; channels are then contiguous per tap (16-byte loads,
 * C % 8 == 0).  Same fp32 summation order over taps, same result. */
HLQ_API int hlq_col2im_ex(const void* dcols, int dtype, int64_t ld, int64_t B, int64_t H, int64_t W,
                          int64_t C, int k, int stride, int pad, int col_order, void* dx_nhwc,
                          int out_dtype, void* stream);

/* Workspace bytes needed by hlq_hq_grad_input / hlq_grad_weight. */
HLQ_API size_t hlq_hq_grad_input_ws(int64_t T, int64_t O, int64_t I);
HLQ_API size_t hlq_grad_weight_ws(int64_t B, int64_t L, int64_t O, int axis, int rank);
/* hlq_grad_weight_ws plus the dW GEMM's split-K / K-chunk slabs: required for
 * contractions past the int32-exact bound (e.g. an 8-bit K > 133,143), which
 * then run as int64-summed chunks up to the reference's MAX_K (quantize.py:21). */
HLQ_API size_t hlq_grad_weight_ws_ex(int64_t B, int64_t L, int64_t O, int64_t I, int axis, int rank, int bits);

/* backprop.py:350-370  hq_grad_input(gy, w, bits): dX (T x I) from gy (T x O)
 * and the fp32 weight W (O x I).  dx_dtype HLQ_F32 with HLQ_EPI_EXACT
 * reproduces the reference bit for bit. */
HLQ_API int hlq_hq_grad_input(const void* gy, int gy_dtype, int64_t T, int64_t O, const float* w, int64_t I,
                      int bits, void* dx, int dx_dtype, int epilogue, void* ws, size_t ws_bytes,
                      void* stream);

/* backprop.py:388-410  hlq_grad_weight(acbp, gy, bits): dW (O x I) from the
 * ACBP payload (K-major, as written by hlq_acbp_compress) and gy (B, L, O).
 * extra is the reference's 1/B (pass 1.0 under a torch mean loss). */
HLQ_API int hlq_grad_weight(const int8_t* payload, int64_t ld_payload, const float* x_scale,
                    const void* gy, int gy_dtype, int64_t B, int64_t L, int64_t O, int64_t I,
                    int axis, uint32_t bitmap, int bits, double extra, void* dw, int dw_dtype,
                    int epilogue, void* ws, size_t ws_bytes, void* stream);

/* Lazy non-finite check (quantize.py:119-120,138-139 raise ValueError on NaN/Inf):
 * every transform entry point ORs 1 into a per-device sticky word when an
 * operand's amax is non-finite.  This copies the word to dst (device or
 * pinned host memory; may be NULL) on `stream` and, with reset, clears it --
 * stream-ordered, no host synchronisation, CUDA-graph capturable. */
HLQ_API int hlq_nonfinite_fetch(uint32_t* dst, int reset, void* stream);

/* Keep n SMs free of libhlq's grids (persistent GEMMs, cooperative transforms);
 * returns the previous value.  For data parallelism: the gradient all-reduce's
 * NCCL kernels (limit them with NCCL_MAX_CTAS) then run beside the HLQ kernels
 * instead of delaying a cooperative transform at its grid barrier. */
HLQ_API int hlq_set_reserved_sms(int n);

#ifdef __cplusplus
}
#endif
#endif /* HLQ_B200_H */
