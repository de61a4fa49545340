// Internal launch declarations shared by the kernel translation units and the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdlib>
#include <cstdint>

namespace hlq {

enum : int { kF32 = 0, kBF16 = 1 };
enum : int { kStats = 0, kQuant = 1, kBoth = 2 };  // kBoth: one cooperative launch
enum : int { kEpiExact = 0, kEpiFast = 1 };

int num_sms();

// Development knob from the environment, read once per process (-1 when unset).
// Launch paths must not call getenv per launch (it scans the environment).
inline int env_knob(const char* name);

// This device's sticky "a quantized operand held NaN/Inf" word (hlq_transform.cu):
// every transform kernel ORs 1 into it when an operand's amax bits are
// non-finite; hlq_nonfinite_fetch copies and resets it (stream-ordered, no
// host sync) so training can check once per step (quantize.py:119-120,138-139).
uint32_t* nonfinite_word();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device, so a process driving several GPUs must set it
// on each.  `done` is the call site's static per-device bitmask.
inline cudaError_t smem_attr_once(const void* kern, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  const unsigned long long bit = 1ull << dev;
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// One pass (STATS or QUANT) of the transform kernels over a (segs x rows x cols)
// view.  do_gx: 16-point HT along cols, codes row-major into dst_gx (row index
// seg*rows + row).  do_gw: projection along rows keeping `bitmap`'s bases,
// codes transposed into dst_gw[col * ld_gw + (seg * nblk + blk) * rank + j].
// stats: {amax_gx, ~minnz_gx, amax_gw, ~minnz_gw} (uint32 bits, max-reduced;
// zero-initialised by the caller before the STATS pass; kBoth also uses
// stats[32] as its grid-barrier counter and stats[64] / stats[96] as its
// per-pass work tickets -- one 128-byte line each -- zero-initialised likewise).  When only do_gw is
// set the gw statistics still live at stats[2..3].
struct TransformArgs {
  const void* src;
  int dtype;
  int64_t segs, rows, cols, ld_src, seg_src;
  bool do_gx, do_gw;
  uint32_t bitmap;
  int bits_gx, bits_gw;
  uint32_t* stats;
  int8_t* dst_gx;
  int64_t ld_gx;
  int8_t* dst_gw;
  int64_t ld_gw;
  float* scale_gx;
  float* scale_gw;
  // optional (kBoth with do_gw): fp32 column sums of the source -> colsum_out,
  // partials in colsum_ws (transform_colsum_ws bytes)
  float* colsum_out = nullptr;
  float* colsum_ws = nullptr;
  // gx codes packed two per byte (low nibble first), ld_gx in bytes (4-bit codes only)
  bool pack_gx = false;
  // stats is a library-owned slot (stats_slot): the fused TMA launch zeroes it
  // again when its last CTA finishes; other launches are preceded by a memset
  bool pooled = false;
};

void launch_transform(const TransformArgs& t, int mode, cudaStream_t stream);
// A fused transform's statistics scratch from the library's per-device ring of
// kStatSlots zero-initialised HLQ_STATS_WS_BYTES slots, for callers that pass
// stats_ws = NULL (no per-launch memset).  A slot is reused kStatSlots fused
// launches later, so fewer than that many may run concurrently on a device.
constexpr int kStatSlots = 64;
uint32_t* stats_slot();
size_t transform_colsum_ws(int64_t segs, int64_t rows, int64_t cols, uint32_t bitmap);
void launch_transform_fallback(const TransformArgs& t, int mode, cudaStream_t stream);

// Conv lowering (hlq_conv.cu).  x is channels-last (B, H, W, C).
void launch_im2col_proj(const void* x, int dtype, int B, int H, int W, int C, int k, int stride,
                        int pad, uint32_t bitmap, int bits, int mode, uint32_t* stats, int8_t* dst,
                        int64_t ld_dst, float* scale, cudaStream_t st);
// The same ACBP on the TMA transform kernel: x read by im2col-mode TMA (one
// 16-pixel x 256-channel tile per tap and step).  Returns false (nothing
// launched) when a tensor map cannot describe x; mode may be kBoth.
bool launch_conv_acbp_tma(const void* x, int dtype, int B, int H, int W, int C, int k, int stride, int pad,
                          uint32_t bitmap, int bits, int mode, uint32_t* stats, int8_t* dst, int64_t ld_dst,
                          float* scale, cudaStream_t stream, bool pooled = false);
// col2im for dcols with (tap, c) column order; false if C % 8 or alignment
// rule out its 16-byte accesses (nothing launched).
bool launch_col2im_tapmajor(const void* dcols, int in_dtype, int64_t ld, int B, int H, int W, int C, int k,
                            int stride, int pad, void* dx, int out_dtype, cudaStream_t st);
void launch_col2im(const void* dcols, int in_dtype, int64_t ld, int B, int H, int W, int C, int k,
                   int stride, int pad, void* dx, int out_dtype, cudaStream_t st);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link dependency).  Returns false if the driver rejects the map.
bool encode_tensor_map(void* map /* CUtensorMap* */, int dtype /* 0 u8, 1 bf16, 2 f32 */,
                       int rank, const void* ptr, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box, int swizzle_128b);

// Returns a cudaError_t-compatible code (0 on success) or -1 if the tensor maps
// could not be encoded.
int launch_gemm_i8(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int64_t M, int64_t N,
                   int64_t K, int64_t groups, int64_t a_gstride, int64_t b_gstride,
                   const float* sa, const float* sb, double extra, int epilogue,
                   void* out, int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc,
                   void* ws, size_t ws_bytes, cudaStream_t stream, int min_splits = 1, bool a4 = false);
// Implicit-GEMM dgrad of a k x k conv with stride s and padding pad: dX (B, H, W, C)
// channels-last = sum over taps and o of G codes (B, Ho, Wo, O; pixel stride
// ldg) at the shifted pixel x W codes (row c*k*k + tap, ld ldw), int32 in TMEM,
// then the dequant epilogue.  s > 1: one launch per output phase (s^2).
int launch_conv_dgrad_i8(const int8_t* G, int64_t ldg, int64_t B, int64_t Ho, int64_t Wo, int64_t O,
                         const int8_t* Wc, int64_t ldw, int64_t C, int k, int stride, int pad, int64_t H,
                         int64_t W, const float* sa, const float* sb, int epilogue, void* out, int out_dtype,
                         int64_t ldo, int32_t* acc_out, int64_t ld_acc, cudaStream_t stream);
// Batched W codes (hlq_weights.cu): Q_bits(HT_O(W_i)) of up to kMaxWeights fp32
// (O_i, I_i) matrices in one cooperative launch; codes_i is (I_i, ld_i) K-major,
// scales_i one fp32.  ws: 8 * n + 8 uint32 (statistics + grid barrier).
constexpr int kMaxWeights = 128;
int launch_weight_codes(int n, const float* const* w, const int64_t* O, const int64_t* I, int bits,
                        int8_t* const* codes, const int64_t* ld, float* const* scales, uint32_t* ws,
                        cudaStream_t stream, void* const* wbf16 = nullptr);
// Two products in one CTA-pair launch (hlq_gemm_i8_multi).
struct GemmDesc {
  const int8_t* A;
  int64_t lda, a_gstride;
  const int8_t* B;
  int64_t ldb, b_gstride;
  int64_t M, N, K, groups;
  const float* sa;
  const float* sb;
  double extra;
  int epilogue;
  void* out;
  int out_dtype;
  int64_t ldo;
  int32_t* acc_out;
  int64_t ld_acc;
  int a4 = 0;  // A packed int4 (lda in bytes of the packed rows)
};
bool gemm_i8_pair2_eligible(const GemmDesc* d);
int launch_gemm_i8_pair2(const GemmDesc* d, cudaStream_t stream);
// True stochastic QUANT pass (hlq_stochastic.cu): along_cols = HT along the
// contiguous axis (codes row-major, ld_dst), else the projection along rows
// (codes K-major per column).  kind: the reference's C-order index of a gw
// element -- 0: (cols, K) transposed, 1: (K, cols), 2: batch axis with
// cols = l2 * o2.  stats from a prior STATS pass.
void launch_stochastic_quant(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols, int64_t ld_src,
                             int64_t seg_src, bool along_cols, uint32_t bitmap, int bits, const uint32_t* stats,
                             int8_t* dst, int64_t ld_dst, float* scale_out, uint64_t k0, uint64_t k1, int kind,
                             int64_t l2, int64_t o2, cudaStream_t st);
// Per-basis sum of |coefficient| of the block transform along rows (calibration).
void launch_basis_energy(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols, int64_t ld_src,
                         int64_t seg_src, double* energy, cudaStream_t st);
// ACBP container (hlq_acbp.cu)
size_t acbp_ws_bytes(int64_t nbytes);
int acbp_pack(const int8_t* codes, int64_t ld, int64_t R, int64_t K, int bits, const uint8_t* head29,
              const float* scale, uint8_t* out, int64_t total, void* ws, cudaStream_t st);
int acbp_check_and_unpack(const uint8_t* buf, int64_t total, int64_t R, int64_t K, int bits, int8_t* codes,
                          int64_t ld, float* scale_out, void* ws, int64_t* bad_offset, bool* crc_ok,
                          cudaStream_t st);
// Baseline-strategy transforms (hlq_baselines.cu): strided view, block FWHT
// along rows keeping `bitmap`'s bases (0 = identity), outputs (s, k, c).
struct XformView {
  const void* src;
  int dtype;
  int64_t segs, rows, cols, nblk;
  int64_t ss, sr, sc;  // source strides (elements)
  uint32_t bitmap;
  int rank;
  int64_t ds, dk, dc;  // destination strides (elements)
  int64_t is, ik, ic;  // reference C-order index strides (stochastic draws)
};
void launch_xform_quant(const XformView& x, int bits, int rounding, uint64_t k0, uint64_t k1, uint32_t* stats,
                        int8_t* dst, float* scale_out, cudaStream_t st);
void launch_xform_f32(const XformView& x, float* dst, cudaStream_t st);
void launch_unproject_f32(const XformView& x, float* dst, cudaStream_t st);
// Workspace bytes that let launch_gemm_i8 split K (0: no split planned).
size_t gemm_i8_ws_bytes(int64_t M, int64_t N, int64_t K, int64_t groups, int min_splits = 1);
// K chunks needed to keep every int32 partial exact: 1 when K * groups * qa * qb < 2^31.
inline int gemm_min_splits(int64_t K, int64_t groups, int qa, int qb) {
  const int64_t kb = (K + 127) / 128 * groups;           // 128-byte K blocks
  const int64_t per = (int64_t(2147483647) / (int64_t(128) * qa * qb));  // blocks per exact chunk
  if (K * groups * int64_t(qa) * qb < int64_t(2147483648LL)) return 1;
  return int((kb + per - 1) / per);
}

inline int env_knob(const char* name) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : -1;
}

}  // namespace hlq
