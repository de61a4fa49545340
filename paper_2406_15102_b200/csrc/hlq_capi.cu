// extern "C" boundary of libhlq_b200.so (declared in include/hlq_b200.h).
// Validation happens here so every failure maps onto one of the reference's
// exception classes; kernels are enqueued on the caller's stream and the
// library never allocates device memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "../../include/hlq_b200.h"
#include "hlq_internal.h"

#define HLQ_VERSION_STRING "hlq_b200 0.1.0 (sm_100a, tcgen05 kind::i8)"

namespace hlq {

// SMs kept free of libhlq's persistent / cooperative grids (hlq_set_reserved_sms):
// under data parallelism the NCCL kernels of the gradient all-reduce run
// concurrently, and a cooperative transform grid sized to every SM would wait
// for them at its grid barrier.
static std::atomic<int> g_reserved_sms{0};

int num_sms() {
  static thread_local int dev_cached = -1;
  static thread_local int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != dev_cached) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
    dev_cached = dev;
  }
  const int avail = sms - g_reserved_sms.load(std::memory_order_relaxed);
  return avail < 2 ? 2 : avail;
}

}  // namespace hlq

extern "C" int hlq_set_reserved_sms(int n) {
  if (n < 0) n = 0;
  return hlq::g_reserved_sms.exchange(n);
}

namespace {

thread_local char g_err[512] = {0};
thread_local int64_t g_err_offset = -1;

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HLQ_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
  return HLQ_OK;
}

inline int64_t pad16(int64_t v) { return (v + 15) & ~int64_t(15); }
inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }
inline int qmax_of(int bits) { return (1 << (bits - 1)) - 1; }

int check_bits(int bits) {
  if (bits != 4 && bits != 8) return fail(HLQ_ERR_PARAMETER, "bits must be 4 or 8, got %d", bits);
  return HLQ_OK;
}
int check_dtype(int dtype) {
  if (dtype != HLQ_F32 && dtype != HLQ_BF16)
    return fail(HLQ_ERR_PARAMETER, "dtype must be HLQ_F32 or HLQ_BF16, got %d", dtype);
  return HLQ_OK;
}
int check_bitmap(uint32_t bitmap) {
  if (bitmap == 0 || bitmap > 0xFFFFu)
    return fail(HLQ_ERR_PARAMETER, "basis bitmap must select 1..16 of 16 bases, got 0x%x", bitmap);
  return HLQ_OK;
}
int check_ld16(int64_t ld, const char* what) {
  if (ld <= 0 || ld % 16 != 0)
    return fail(HLQ_ERR_PARAMETER, "%s leading dimension must be a positive multiple of 16, got %lld",
                what, (long long)ld);
  return HLQ_OK;
}

#define HLQ_TRY(expr)          \
  do {                         \
    int _s = (expr);           \
    if (_s != HLQ_OK) return _s; \
  } while (0)

int proj_rows_checked(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                      int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits, int8_t* dst,
                      int64_t ld_dst) {
  HLQ_TRY(check_dtype(dtype));
  HLQ_TRY(check_bits(bits));
  HLQ_TRY(check_bitmap(bitmap));
  if (segs < 0 || rows < 0 || cols < 0 || ld_src < cols || (segs > 1 && seg_src < rows * ld_src))
    return fail(HLQ_ERR_DIMENSION, "bad projection view segs=%lld rows=%lld cols=%lld ld=%lld",
                (long long)segs, (long long)rows, (long long)cols, (long long)ld_src);
  const int64_t k = segs * ((rows + 15) / 16) * __builtin_popcount(bitmap);
  if (dst) {
    HLQ_TRY(check_ld16(ld_dst, "projection output"));
    if (ld_dst < k)
      return fail(HLQ_ERR_DIMENSION, "projection output ld %lld < K %lld", (long long)ld_dst,
                  (long long)k);
  }
  if (!src && segs * rows * cols > 0) return fail(HLQ_ERR_PARAMETER, "null source");
  return HLQ_OK;
}

}  // namespace

extern "C" {

const char* hlq_version(void) { return HLQ_VERSION_STRING; }
const char* hlq_last_error(void) { return g_err; }

int hlq_device_ok(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10 ? 1 : 0;
}

// stats_ws == NULL: a library-owned, self-cleaning statistics slot (no memset
// launch); otherwise the caller's scratch, zeroed here
static void prepare_stats(hlq::TransformArgs& t, uint32_t* stats_ws, cudaStream_t st) {
  if (stats_ws) {
    t.stats = stats_ws;
    cudaMemsetAsync(stats_ws, 0, HLQ_STATS_WS_BYTES, st);
  } else {
    t.stats = hlq::stats_slot();
    t.pooled = true;
  }
}

int hlq_quantize_ht_cols(const void* src, int dtype, int64_t rows, int64_t cols, int64_t ld_src,
                         int bits, uint32_t* stats_ws, int8_t* dst, int64_t ld_dst,
                         float* scale_out, void* stream) {
  HLQ_TRY(check_dtype(dtype));
  HLQ_TRY(check_bits(bits));
  HLQ_TRY(check_ld16(ld_dst, "codes"));
  if (rows < 0 || cols < 0 || ld_src < cols || ld_dst < pad16(cols))
    return fail(HLQ_ERR_DIMENSION, "bad ht_cols view rows=%lld cols=%lld ld_src=%lld ld_dst=%lld",
                (long long)rows, (long long)cols, (long long)ld_src, (long long)ld_dst);
  if (!src && rows * cols > 0) return fail(HLQ_ERR_PARAMETER, "null source");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  hlq::TransformArgs t{};
  t.src = src; t.dtype = dtype; t.segs = 1; t.rows = rows; t.cols = cols; t.ld_src = ld_src;
  t.seg_src = rows * ld_src; t.do_gx = true; t.do_gw = false; t.bitmap = 0xFFFF;
  t.bits_gx = bits; t.bits_gw = bits; t.stats = stats_ws; t.dst_gx = dst; t.ld_gx = ld_dst;
  t.scale_gx = scale_out;
  prepare_stats(t, stats_ws, st);
  hlq::launch_transform(t, hlq::kBoth, st);
  return cuda_status("hlq_quantize_ht_cols");
}

static hlq::TransformArgs proj_args(const void* src, int dtype, int64_t segs, int64_t rows,
                                    int64_t cols, int64_t ld_src, int64_t seg_src, uint32_t bitmap,
                                    int bits, uint32_t* stats, int8_t* dst, int64_t ld_dst,
                                    float* scale_out) {
  hlq::TransformArgs t{};
  t.src = src; t.dtype = dtype; t.segs = segs; t.rows = rows; t.cols = cols; t.ld_src = ld_src;
  t.seg_src = seg_src; t.do_gx = false; t.do_gw = true; t.bitmap = bitmap; t.bits_gx = bits;
  t.bits_gw = bits; t.stats = stats; t.dst_gw = dst; t.ld_gw = ld_dst; t.scale_gw = scale_out;
  return t;
}

int hlq_proj_rows_amax(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                       int64_t ld_src, int64_t seg_src, uint32_t bitmap, uint32_t* stats,
                       void* stream) {
  HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, 8, nullptr, 0));
  hlq::launch_transform(proj_args(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, 8, stats,
                                  nullptr, 0, nullptr),
                        hlq::kStats, static_cast<cudaStream_t>(stream));
  return cuda_status("hlq_proj_rows_amax");
}

int hlq_proj_rows_quant(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                        int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits,
                        const uint32_t* stats, int8_t* dst, int64_t ld_dst, float* scale_out,
                        void* stream) {
  HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits, dst, ld_dst));
  hlq::launch_transform(proj_args(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits,
                                  const_cast<uint32_t*>(stats), dst, ld_dst, scale_out),
                        hlq::kQuant, static_cast<cudaStream_t>(stream));
  return cuda_status("hlq_proj_rows_quant");
}

int hlq_quantize_proj_rows(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                           int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits,
                           uint32_t* stats_ws, int8_t* dst, int64_t ld_dst, float* scale_out,
                           void* stream) {
  HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits, dst, ld_dst));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  hlq::TransformArgs t = proj_args(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits,
                                   stats_ws, dst, ld_dst, scale_out);
  prepare_stats(t, stats_ws, st);
  hlq::launch_transform(t, hlq::kBoth, st);
  return cuda_status("hlq_quantize_proj_rows");
}

int hlq_transform_pass(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                       int64_t ld_src, int64_t seg_src, int do_gx, int do_gw, uint32_t bitmap,
                       int bits_gx, int bits_gw, int mode, uint32_t* stats, int8_t* dst_gx,
                       int64_t ld_gx, int8_t* dst_gw, int64_t ld_gw, float* scale_gx,
                       float* scale_gw, void* stream) {
  if (!do_gx && !do_gw) return fail(HLQ_ERR_PARAMETER, "transform pass with neither operand");
  if (mode != 0 && mode != 1) return fail(HLQ_ERR_PARAMETER, "mode must be 0 (stats) or 1 (quant)");
  HLQ_TRY(check_bits(bits_gx));
  HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, do_gw ? bitmap : 0xFFFF,
                            bits_gw, mode == 1 && do_gw ? dst_gw : nullptr, ld_gw));
  if (do_gx && mode == 1) {
    HLQ_TRY(check_ld16(ld_gx, "gx codes"));
    if (ld_gx < pad16(cols)) return fail(HLQ_ERR_DIMENSION, "gx codes ld < pad16(cols)");
  }
  hlq::TransformArgs t = proj_args(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits_gw,
                                   stats, dst_gw, ld_gw, scale_gw);
  t.do_gx = do_gx != 0; t.do_gw = do_gw != 0; t.bits_gx = bits_gx; t.dst_gx = dst_gx;
  t.ld_gx = ld_gx; t.scale_gx = scale_gx;
  hlq::launch_transform(t, mode, static_cast<cudaStream_t>(stream));
  return cuda_status("hlq_transform_pass");
}

int hlq_quantize_dual(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                      int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits_gx, int bits_gw,
                      uint32_t* stats_ws, int8_t* dst_gx, int64_t ld_gx, int8_t* dst_gw,
                      int64_t ld_gw, float* scale_gx, float* scale_gw, void* stream) {
  HLQ_TRY(check_bits(bits_gx));
  HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits_gw, dst_gw,
                            ld_gw));
  HLQ_TRY(check_ld16(ld_gx, "gx codes"));
  if (ld_gx < pad16(cols)) return fail(HLQ_ERR_DIMENSION, "gx codes ld < pad16(cols)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  hlq::TransformArgs t = proj_args(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits_gw,
                                   stats_ws, dst_gw, ld_gw, scale_gw);
  t.do_gx = true; t.bits_gx = bits_gx; t.dst_gx = dst_gx; t.ld_gx = ld_gx; t.scale_gx = scale_gx;
  prepare_stats(t, stats_ws, st);
  hlq::launch_transform(t, hlq::kBoth, st);
  return cuda_status("hlq_quantize_dual");
}

size_t hlq_quantize_dual_colsum_ws(int64_t segs, int64_t rows, int64_t cols, uint32_t bitmap) {
  return hlq::transform_colsum_ws(segs, rows, cols, bitmap);
}

int hlq_quantize_dual_colsum(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                             int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits_gx, int bits_gw,
                             uint32_t* stats_ws, int8_t* dst_gx, int64_t ld_gx, int8_t* dst_gw, int64_t ld_gw,
                             float* scale_gx, float* scale_gw, float* colsum_out, void* colsum_ws,
                             size_t colsum_ws_bytes, void* stream) {
  HLQ_TRY(check_bits(bits_gx));
  HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits_gw, dst_gw,
                            ld_gw));
  HLQ_TRY(check_ld16(ld_gx, "gx codes"));
  if (ld_gx < pad16(cols)) return fail(HLQ_ERR_DIMENSION, "gx codes ld < pad16(cols)");
  if (!colsum_out) return fail(HLQ_ERR_PARAMETER, "null column-sum output");
  const size_t need = hlq::transform_colsum_ws(segs, rows, cols, bitmap);
  if (colsum_ws_bytes < need || (need && !colsum_ws))
    return fail(HLQ_ERR_PARAMETER, "column-sum workspace needs %zu bytes, got %zu", need, colsum_ws_bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  hlq::TransformArgs t = proj_args(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits_gw,
                                   stats_ws, dst_gw, ld_gw, scale_gw);
  t.do_gx = true; t.bits_gx = bits_gx; t.dst_gx = dst_gx; t.ld_gx = ld_gx; t.scale_gx = scale_gx;
  t.colsum_out = colsum_out;
  t.colsum_ws = static_cast<float*>(colsum_ws);
  prepare_stats(t, stats_ws, st);
  hlq::launch_transform(t, hlq::kBoth, st);
  return cuda_status("hlq_quantize_dual_colsum");
}

int hlq_quantize_dual_ex(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols, int64_t ld_src,
                         int64_t seg_src, uint32_t bitmap, int bits_gx, int bits_gw, uint32_t* stats_ws,
                         void* dst_gx, int64_t ld_gx, int pack_gx, int8_t* dst_gw, int64_t ld_gw, float* scale_gx,
                         float* scale_gw, float* colsum_out, void* colsum_ws, size_t colsum_ws_bytes,
                         void* stream) {
  HLQ_TRY(check_bits(bits_gx));
  HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits_gw, dst_gw,
                            ld_gw));
  HLQ_TRY(check_ld16(ld_gx, "gx codes"));
  if (pack_gx && bits_gx != 4) return fail(HLQ_ERR_PARAMETER, "packed gx codes are 4-bit, got bits_gx=%d", bits_gx);
  if (ld_gx < (pack_gx ? pad16(cols) / 2 : pad16(cols)))
    return fail(HLQ_ERR_DIMENSION, "gx codes ld %lld too small for %lld columns", (long long)ld_gx, (long long)cols);
  if (colsum_out) {
    const size_t need = hlq::transform_colsum_ws(segs, rows, cols, bitmap);
    if (colsum_ws_bytes < need || (need && !colsum_ws))
      return fail(HLQ_ERR_PARAMETER, "column-sum workspace needs %zu bytes, got %zu", need, colsum_ws_bytes);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  hlq::TransformArgs t = proj_args(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits_gw,
                                   stats_ws, dst_gw, ld_gw, scale_gw);
  t.do_gx = true; t.bits_gx = bits_gx; t.dst_gx = static_cast<int8_t*>(dst_gx); t.ld_gx = ld_gx;
  t.scale_gx = scale_gx; t.pack_gx = pack_gx != 0;
  t.colsum_out = colsum_out;
  t.colsum_ws = static_cast<float*>(colsum_ws);
  prepare_stats(t, stats_ws, st);
  hlq::launch_transform(t, hlq::kBoth, st);
  return cuda_status("hlq_quantize_dual_ex");
}

int hlq_gemm_i8(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int64_t M, int64_t N,
                int64_t K, int bits_a, int bits_b, const float* sa, const float* sb, double extra,
                int epilogue, void* out, int out_dtype, int64_t ldo, int32_t* acc_out,
                int64_t ld_acc, void* stream) {
  return hlq_gemm_i8_grouped(A, lda, lda * M, B, ldb, ldb * N, M, N, K, 1, bits_a, bits_b, sa, sb,
                             extra, epilogue, out, out_dtype, ldo, acc_out, ld_acc, stream);
}

int hlq_gemm_i8_grouped(const int8_t* A, int64_t lda, int64_t a_gstride, const int8_t* B,
                        int64_t ldb, int64_t b_gstride, int64_t M, int64_t N, int64_t K,
                        int64_t groups, int bits_a, int bits_b, const float* sa, const float* sb,
                        double extra, int epilogue, void* out, int out_dtype, int64_t ldo,
                        int32_t* acc_out, int64_t ld_acc, void* stream) {
  return hlq_gemm_i8_ex(A, lda, a_gstride, B, ldb, b_gstride, M, N, K, groups, bits_a, bits_b, sa, sb,
                        extra, epilogue, out, out_dtype, ldo, acc_out, ld_acc, nullptr, 0, stream);
}

static int gemm_ex_impl(const int8_t* A, int64_t lda, int64_t a_gstride, const int8_t* B, int64_t ldb,
                   int64_t b_gstride, int64_t M, int64_t N, int64_t K, int64_t groups, int bits_a,
                   int bits_b, const float* sa, const float* sb, double extra, int epilogue, void* out,
                   int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc, void* ws,
                   size_t ws_bytes, void* stream, bool a4);

int hlq_gemm_i8_multi(int n, const hlq_gemm_desc* d, void* stream) {
  if (n < 1 || n > 2 || !d) return fail(HLQ_ERR_PARAMETER, "hlq_gemm_i8_multi takes 1 or 2 products, got %d", n);
  bool fuse = n == 2;
  for (int q = 0; q < n; ++q) {
    const hlq_gemm_desc& g = d[q];
    // validate each product exactly as the single call does (zero-sized products skip the launch)
    if (g.M == 0 || g.N == 0 || (g.groups > 1) || g.acc_out || !g.out) fuse = false;
  }
  if (fuse) {
    for (int q = 0; q < 2; ++q) {
      const hlq_gemm_desc& g = d[q];
      HLQ_TRY(check_bits(g.bits_a));
      HLQ_TRY(check_bits(g.bits_b));
      HLQ_TRY(check_dtype(g.out_dtype));
      HLQ_TRY(check_ld16(g.lda, "A"));
      HLQ_TRY(check_ld16(g.ldb, "B"));
      if (g.a_packed && g.bits_a != 4) return fail(HLQ_ERR_PARAMETER, "packed A holds 4-bit codes");
      if (g.M < 0 || g.N < 0 || g.K <= 0 || g.lda < (g.a_packed ? (g.K + 1) / 2 : g.K) || g.ldb < g.K || g.ldo < g.N || g.M > INT32_MAX ||
          g.N > INT32_MAX || g.K > INT32_MAX)
        return fail(HLQ_ERR_DIMENSION, "bad GEMM shape M=%lld N=%lld K=%lld", (long long)g.M, (long long)g.N,
                    (long long)g.K);
      if ((long double)g.K * qmax_of(g.bits_a) * qmax_of(g.bits_b) >= 2147483648.0L)
        return fail(HLQ_ERR_PARAMETER, "contraction extent %lld exceeds the int32-exact bound", (long long)g.K);
      if (g.epilogue != HLQ_EPI_EXACT && g.epilogue != HLQ_EPI_FAST)
        return fail(HLQ_ERR_PARAMETER, "unknown epilogue %d", g.epilogue);
    }
    hlq::GemmDesc gd[2];
    for (int q = 0; q < 2; ++q) {
      const hlq_gemm_desc& g = d[q];
      gd[q] = hlq::GemmDesc{g.A, g.lda, g.lda * g.M, g.B, g.ldb, g.ldb * g.N, g.M, g.N, g.K, 1, g.sa, g.sb,
                            g.extra, g.epilogue, g.out, g.out_dtype, g.ldo, nullptr, 0, g.a_packed ? 1 : 0};
    }
    if (hlq::gemm_i8_pair2_eligible(gd)) {
      int e = hlq::launch_gemm_i8_pair2(gd, static_cast<cudaStream_t>(stream));
      if (e == -1) return fail(HLQ_ERR_CUDA, "cuTensorMapEncodeTiled rejected the operands");
      if (e != 0) return fail(HLQ_ERR_CUDA, "hlq_gemm_i8_multi: %s", cudaGetErrorString(cudaError_t(e)));
      return HLQ_OK;
    }
  }
  for (int q = 0; q < n; ++q) {
    const hlq_gemm_desc& g = d[q];
    HLQ_TRY(gemm_ex_impl(g.A, g.lda, g.a_gstride, g.B, g.ldb, g.b_gstride, g.M, g.N, g.K, g.groups, g.bits_a,
                         g.bits_b, g.sa, g.sb, g.extra, g.epilogue, g.out, g.out_dtype, g.ldo, g.acc_out, g.ld_acc,
                         nullptr, 0, stream, g.a_packed != 0));
  }
  return HLQ_OK;
}

int hlq_nonfinite_fetch(uint32_t* dst, int reset, void* stream) {
  uint32_t* w = hlq::nonfinite_word();
  if (!w) return fail(HLQ_ERR_CUDA, "non-finite flag unavailable on this device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dst && cudaMemcpyAsync(dst, w, sizeof(uint32_t), cudaMemcpyDefault, st) != cudaSuccess)
    return cuda_status("hlq_nonfinite_fetch");
  if (reset && cudaMemsetAsync(w, 0, sizeof(uint32_t), st) != cudaSuccess) return cuda_status("hlq_nonfinite_fetch");
  return HLQ_OK;
}

size_t hlq_gemm_i8_ws(int64_t M, int64_t N, int64_t K, int64_t groups) {
  if (M <= 0 || N <= 0 || K <= 0 || groups < 1) return 0;
  return hlq::gemm_i8_ws_bytes(M, N, K, groups);
}

size_t hlq_gemm_i8_ws_bits(int64_t M, int64_t N, int64_t K, int64_t groups, int bits_a, int bits_b) {
  if (M <= 0 || N <= 0 || K <= 0 || groups < 1 || check_bits(bits_a) || check_bits(bits_b)) return 0;
  return hlq::gemm_i8_ws_bytes(M, N, K, groups,
                               hlq::gemm_min_splits(K, groups, qmax_of(bits_a), qmax_of(bits_b)));
}

// int_matmul's advertised bound (quantize.py:21,166-170): MAX_K = {8: 10^6, 4: 10^7}
static int64_t max_k_of(int bits) { return bits == 8 ? 1000000 : 10000000; }

static int gemm_ex_impl(const int8_t* A, int64_t lda, int64_t a_gstride, const int8_t* B, int64_t ldb,
                   int64_t b_gstride, int64_t M, int64_t N, int64_t K, int64_t groups, int bits_a,
                   int bits_b, const float* sa, const float* sb, double extra, int epilogue, void* out,
                   int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc, void* ws,
                   size_t ws_bytes, void* stream, bool a4) {
  if (groups < 1 || groups > 65535 || (groups > 1 && (a_gstride % 16 || b_gstride % 16 ||
                                                      a_gstride < lda * M || b_gstride < ldb * N)))
    return fail(HLQ_ERR_PARAMETER, "bad K-group layout groups=%lld", (long long)groups);
  HLQ_TRY(check_bits(bits_a));
  HLQ_TRY(check_bits(bits_b));
  HLQ_TRY(check_dtype(out_dtype));
  HLQ_TRY(check_ld16(lda, "A"));
  if (a4 && bits_a != 4) return fail(HLQ_ERR_PARAMETER, "packed A holds 4-bit codes, got bits_a=%d", bits_a);
  // the widened packed codes are 16 * code: the int32 accumulator holds 16 x the sum
  if (a4 && (long double)K * groups * 16 * 7 * qmax_of(bits_b) >= 2147483648.0L)
    return fail(HLQ_ERR_PARAMETER, "packed-A contraction extent %lld exceeds the int32-exact bound", (long long)K);
  const int64_t a_row = a4 ? (K + 1) / 2 : K;  // bytes of one A row
  HLQ_TRY(check_ld16(ldb, "B"));
  if (M < 0 || N < 0 || K <= 0 || lda < a_row || ldb < K || (out && ldo < N) || (acc_out && ld_acc < N))
    return fail(HLQ_ERR_DIMENSION, "bad GEMM shape M=%lld N=%lld K=%lld", (long long)M, (long long)N,
                (long long)K);
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
    return fail(HLQ_ERR_DIMENSION, "GEMM extent exceeds int32");
  const int64_t kbound = max_k_of(bits_a) < max_k_of(bits_b) ? max_k_of(bits_a) : max_k_of(bits_b);
  if (K * groups > kbound)
    return fail(HLQ_ERR_PARAMETER, "contraction extent %lld exceeds the overflow-safe bound %lld for %dx%d-bit operands",
                (long long)(K * groups), (long long)kbound, bits_a, bits_b);
  const int min_splits = hlq::gemm_min_splits(K, groups, qmax_of(bits_a), qmax_of(bits_b));
  if (min_splits > 1) {
    // past the int32-exact bound: int32 chunks summed in int64 (needs the chunk slabs)
    if (acc_out)
      return fail(HLQ_ERR_PARAMETER, "contraction extent %lld exceeds the int32 accumulator dump bound",
                  (long long)(K * groups));
    if (!ws || ws_bytes < hlq::gemm_i8_ws_bytes(M, N, K, groups, min_splits))
      return fail(HLQ_ERR_PARAMETER, "contraction extent %lld needs K chunks: hlq_gemm_i8_ws_bits bytes of workspace",
                  (long long)(K * groups));
  }
  if (epilogue != HLQ_EPI_EXACT && epilogue != HLQ_EPI_FAST)
    return fail(HLQ_ERR_PARAMETER, "unknown epilogue %d", epilogue);
  if (M == 0 || N == 0) return HLQ_OK;
  int e = hlq::launch_gemm_i8(A, lda, B, ldb, M, N, K, groups, a_gstride, b_gstride, sa, sb, extra,
                              epilogue, out, out_dtype, ldo, acc_out, ld_acc, ws, ws_bytes,
                              static_cast<cudaStream_t>(stream), min_splits, a4);
  if (e == -2) return fail(HLQ_ERR_PARAMETER, "long contraction: output / workspace not 16-byte aligned");
  if (e == -1) return fail(HLQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable or rejected the operands");
  if (e != 0) return fail(HLQ_ERR_CUDA, "hlq_gemm_i8: %s", cudaGetErrorString(cudaError_t(e)));
  return HLQ_OK;
}

int hlq_gemm_i8_ex(const int8_t* A, int64_t lda, int64_t a_gstride, const int8_t* B, int64_t ldb,
                   int64_t b_gstride, int64_t M, int64_t N, int64_t K, int64_t groups, int bits_a,
                   int bits_b, const float* sa, const float* sb, double extra, int epilogue, void* out,
                   int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc, void* ws,
                   size_t ws_bytes, void* stream) {
  return gemm_ex_impl(A, lda, a_gstride, B, ldb, b_gstride, M, N, K, groups, bits_a, bits_b, sa, sb, extra,
                      epilogue, out, out_dtype, ldo, acc_out, ld_acc, ws, ws_bytes, stream, false);
}

int hlq_gemm_i4a_ex(const uint8_t* A, int64_t lda, int64_t a_gstride, const int8_t* B, int64_t ldb,
                    int64_t b_gstride, int64_t M, int64_t N, int64_t K, int64_t groups, int bits_b,
                    const float* sa, const float* sb, double extra, int epilogue, void* out, int out_dtype,
                    int64_t ldo, void* ws, size_t ws_bytes, void* stream) {
  return gemm_ex_impl(reinterpret_cast<const int8_t*>(A), lda, a_gstride, B, ldb, b_gstride, M, N, K, groups, 4,
                      bits_b, sa, sb, extra, epilogue, out, out_dtype, ldo, nullptr, 0, ws, ws_bytes, stream, true);
}

size_t hlq_quantize_weights_ws(int n) { return n < 0 ? 0 : size_t(8 * n + 8) * sizeof(uint32_t); }

int hlq_quantize_weights(int n, const float* const* w, const int64_t* O, const int64_t* I, int bits,
                         int8_t* const* codes, const int64_t* ld, float* const* scales, uint32_t* ws,
                         size_t ws_bytes, void* stream) {
  return hlq_quantize_weights_ex(n, w, O, I, bits, codes, ld, scales, nullptr, ws, ws_bytes, stream);
}

int hlq_quantize_weights_ex(int n, const float* const* w, const int64_t* O, const int64_t* I, int bits,
                            int8_t* const* codes, const int64_t* ld, float* const* scales, void* const* wbf16,
                            uint32_t* ws, size_t ws_bytes, void* stream) {
  HLQ_TRY(check_bits(bits));
  if (n < 0 || n > hlq::kMaxWeights)
    return fail(HLQ_ERR_PARAMETER, "batched weight codes take 0..%d tensors, got %d", hlq::kMaxWeights, n);
  if (n == 0) return HLQ_OK;
  if (ws_bytes < hlq_quantize_weights_ws(n)) return fail(HLQ_ERR_PARAMETER, "workspace too small");
  for (int i = 0; i < n; ++i) {
    if (!w[i] || !codes[i] || O[i] <= 0 || I[i] <= 0 || O[i] > INT32_MAX / 2 || I[i] > INT32_MAX / 2)
      return fail(HLQ_ERR_DIMENSION, "weight %d: bad shape or null pointer", i);
    HLQ_TRY(check_ld16(ld[i], "weight codes"));
    if (ld[i] < pad16(O[i]))
      return fail(HLQ_ERR_DIMENSION, "weight %d: codes ld %lld < pad16(O) %lld", i, (long long)ld[i],
                  (long long)pad16(O[i]));
    if (reinterpret_cast<uintptr_t>(codes[i]) % 16) return fail(HLQ_ERR_PARAMETER, "codes %d not 16-byte aligned", i);
  }
  int e = hlq::launch_weight_codes(n, w, O, I, bits, codes, ld, scales, ws, static_cast<cudaStream_t>(stream),
                                   wbf16);
  if (e != 0) return fail(HLQ_ERR_CUDA, "hlq_quantize_weights: %s", cudaGetErrorString(cudaError_t(e)));
  return cuda_status("hlq_quantize_weights");
}

int hlq_quantize_stochastic(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                            int64_t ld_src, int64_t seg_src, int along_cols, uint32_t bitmap, int bits,
                            uint64_t seed, uint64_t counter, int index_kind, int64_t l2, int64_t o2,
                            uint32_t* stats_ws, int8_t* dst, int64_t ld_dst, float* scale_out, void* stream) {
  HLQ_TRY(check_dtype(dtype));
  HLQ_TRY(check_bits(bits));
  if (index_kind < 0 || index_kind > 2) return fail(HLQ_ERR_PARAMETER, "index_kind must be 0, 1 or 2");
  if (along_cols) {
    HLQ_TRY(check_ld16(ld_dst, "codes"));
    if (segs < 0 || rows < 0 || cols < 0 || ld_src < cols || ld_dst < pad16(cols) ||
        (segs > 1 && seg_src < rows * ld_src))
      return fail(HLQ_ERR_DIMENSION, "bad stochastic view");
  } else {
    HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, bitmap, bits, dst, ld_dst));
    if (index_kind == 2 && (l2 <= 0 || o2 <= 0 || l2 * o2 != cols))
      return fail(HLQ_ERR_DIMENSION, "batch-axis index layout needs cols == l2 * o2");
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  hlq::TransformArgs t = proj_args(src, dtype, segs, rows, cols, ld_src, seg_src, along_cols ? 0xFFFFu : bitmap,
                                   bits, stats_ws, nullptr, 0, nullptr);
  t.do_gx = along_cols != 0;
  t.do_gw = along_cols == 0;
  t.bits_gx = bits;
  cudaMemsetAsync(stats_ws, 0, HLQ_STATS_WS_BYTES, st);
  hlq::launch_transform(t, hlq::kStats, st);  // statistics do not depend on the rounding
  hlq::launch_stochastic_quant(src, dtype, segs, rows, cols, ld_src, seg_src, along_cols != 0, bitmap, bits,
                               along_cols ? stats_ws : stats_ws + 2, dst, ld_dst, scale_out, seed, counter,
                               index_kind, l2, o2, st);
  return cuda_status("hlq_quantize_stochastic");
}

int hlq_basis_energy(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols, int64_t ld_src,
                     int64_t seg_src, double* energy16, void* stream) {
  HLQ_TRY(proj_rows_checked(src, dtype, segs, rows, cols, ld_src, seg_src, 0xFFFFu, 8, nullptr, 0));
  if (!energy16) return fail(HLQ_ERR_PARAMETER, "null energy output");
  hlq::launch_basis_energy(src, dtype, segs, rows, cols, ld_src, seg_src, energy16, static_cast<cudaStream_t>(stream));
  return cuda_status("hlq_basis_energy");
}

static int xform_view(const hlq_xform* v, bool quant_source_dtype, hlq::XformView* x) {
  if (!v) return fail(HLQ_ERR_PARAMETER, "null view");
  if (quant_source_dtype) HLQ_TRY(check_dtype(v->src_dtype));
  if (v->segs < 0 || v->rows < 0 || v->cols < 0) return fail(HLQ_ERR_DIMENSION, "negative view extent");
  if (!v->src && v->segs * v->rows * v->cols > 0) return fail(HLQ_ERR_PARAMETER, "null source");
  if (v->bitmap > 0xFFFFu) return fail(HLQ_ERR_PARAMETER, "bitmap has bits above the 16-point block");
  *x = hlq::XformView{};
  x->src = v->src; x->dtype = quant_source_dtype ? v->src_dtype : HLQ_F32;
  x->segs = v->segs; x->rows = v->rows; x->cols = v->cols; x->nblk = (v->rows + 15) / 16;
  x->ss = v->src_stride[0]; x->sr = v->src_stride[1]; x->sc = v->src_stride[2];
  x->bitmap = v->bitmap; x->rank = __builtin_popcount(v->bitmap);
  x->ds = v->dst_stride[0]; x->dk = v->dst_stride[1]; x->dc = v->dst_stride[2];
  x->is = v->idx_stride[0]; x->ik = v->idx_stride[1]; x->ic = v->idx_stride[2];
  return HLQ_OK;
}

int hlq_xform_quantize(const hlq_xform* view, int bits, int rounding, uint64_t seed, uint64_t counter,
                       uint32_t* stats_ws, int8_t* dst, float* scale_out, void* stream) {
  hlq::XformView x;
  HLQ_TRY(xform_view(view, true, &x));
  HLQ_TRY(check_bits(bits));
  if (rounding != 0 && rounding != 1) return fail(HLQ_ERR_PARAMETER, "rounding must be 0 (pseudo) or 1 (stochastic)");
  if (!stats_ws || !scale_out) return fail(HLQ_ERR_PARAMETER, "null stats or scale");
  if (!dst && x.segs * x.rows * x.cols > 0) return fail(HLQ_ERR_PARAMETER, "null codes");
  hlq::launch_xform_quant(x, bits, rounding, seed, counter, stats_ws, dst, scale_out, static_cast<cudaStream_t>(stream));
  return cuda_status("hlq_xform_quantize");
}

int hlq_xform_project_f32(const hlq_xform* view, float* dst, void* stream) {
  hlq::XformView x;
  HLQ_TRY(xform_view(view, true, &x));
  if (!dst && x.segs * x.rows * x.cols > 0) return fail(HLQ_ERR_PARAMETER, "null output");
  if (x.segs * x.rows * x.cols == 0) return HLQ_OK;
  hlq::launch_xform_f32(x, dst, static_cast<cudaStream_t>(stream));
  return cuda_status("hlq_xform_project_f32");
}

int hlq_xform_unproject_f32(const hlq_xform* view, float* dst, void* stream) {
  hlq::XformView x;
  HLQ_TRY(xform_view(view, false, &x));
  if (x.bitmap == 0) return fail(HLQ_ERR_PARAMETER, "unproject needs at least one kept basis");
  if (!dst && x.segs * x.rows * x.cols > 0) return fail(HLQ_ERR_PARAMETER, "null output");
  if (x.segs * x.rows * x.cols == 0) return HLQ_OK;
  hlq::launch_unproject_f32(x, dst, static_cast<cudaStream_t>(stream));
  return cuda_status("hlq_xform_unproject_f32");
}

int64_t hlq_acbp_container_bytes(int64_t rows, int64_t k, int bits) {
  const int64_t count = rows * k;
  return 33 + (bits == 8 ? count : (count + 1) / 2) + 4;
}

size_t hlq_acbp_ws(int64_t total_bytes) { return hlq::acbp_ws_bytes(total_bytes < 0 ? 0 : total_bytes); }

int64_t hlq_last_error_offset(void) { return g_err_offset; }

static int ffail(int64_t offset, const char* fmt, ...) {
  char msg[400];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(msg, sizeof(msg), fmt, ap);
  va_end(ap);
  g_err_offset = offset;
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return HLQ_ERR_FORMAT;
}

// acbp.py:_container_axis + projected_shape, in our K-major terms
static void container_geometry(int64_t B, int64_t L, int64_t I, int block, int rank, int* axis, int64_t* rows,
                               int64_t* k) {
  int ax;
  if (L >= block || B >= block) ax = L >= block ? 1 : 0;
  else ax = L >= B ? 1 : 0;
  *axis = ax;
  if (ax == 1) {
    *rows = I;
    *k = B * ((L + block - 1) / block) * rank;
  } else {
    *rows = L * I;
    *k = ((B + block - 1) / block) * rank;
  }
}

int hlq_acbp_pack(const int8_t* payload, int64_t ld, int64_t rows, int64_t k, int bits, int block,
                  uint32_t bitmap, int64_t B, int64_t L, int64_t I, const float* scale, uint8_t* out,
                  int64_t out_bytes, void* ws, size_t ws_bytes, void* stream) {
  HLQ_TRY(check_bits(bits));
  const int rank = __builtin_popcount(bitmap);
  if (block != 2 && block != 4 && block != 8 && block != 16)
    return fail(HLQ_ERR_PARAMETER, "container format supports block sizes 2..16, got %d", block);
  if (bitmap == 0 || (bitmap >> block)) return fail(HLQ_ERR_PARAMETER, "bad basis bitmap 0x%x", bitmap);
  if (B < 0 || L < 0 || I < 0 || B > UINT32_MAX || L > UINT32_MAX || I > UINT32_MAX)
    return fail(HLQ_ERR_DIMENSION, "shape does not fit the container's u32 dims");
  int axis;
  int64_t rr, kk;
  container_geometry(B, L, I, block, rank, &axis, &rr, &kk);
  if (rr != rows || kk != k)
    return fail(HLQ_ERR_PARAMETER, "payload geometry (%lld x %lld) is inconsistent with the container axis rule "
                "(%lld x %lld)", (long long)rows, (long long)k, (long long)rr, (long long)kk);
  if (rows * k > 0 && ld < k) return fail(HLQ_ERR_DIMENSION, "payload ld < K");
  const int64_t total = hlq_acbp_container_bytes(rows, k, bits);
  if (out_bytes != total) return fail(HLQ_ERR_DIMENSION, "container buffer must be %lld bytes", (long long)total);
  if (ws_bytes < hlq_acbp_ws(total)) return fail(HLQ_ERR_PARAMETER, "workspace too small");
  uint8_t h[29];
  memcpy(h, "ACBP", 4);
  const uint16_t ver = 1, rk = uint16_t(rank), bm = uint16_t(bitmap);
  memcpy(h + 4, &ver, 2);
  h[6] = uint8_t(bits);
  h[7] = uint8_t(block);
  memcpy(h + 8, &rk, 2);
  memcpy(h + 10, &bm, 2);
  h[12] = 3;
  const uint32_t dims[3] = {uint32_t(B), uint32_t(L), uint32_t(I)}, ns = 1;
  memcpy(h + 13, dims, 12);
  memcpy(h + 25, &ns, 4);
  const int e = hlq::acbp_pack(payload, ld, rows, k, bits, h, scale, out, total, ws, static_cast<cudaStream_t>(stream));
  if (e) return fail(HLQ_ERR_CUDA, "hlq_acbp_pack: %s", cudaGetErrorString(cudaError_t(e)));
  return HLQ_OK;
}

int hlq_acbp_parse(const uint8_t* buf, int64_t nbytes, hlq_acbp_info* info, void* stream) {
  uint8_t h[33] = {0};
  const int64_t n = nbytes < 33 ? nbytes : 33;
  if (n > 0) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaMemcpyAsync(h, buf, size_t(n), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_status("hlq_acbp_parse");
  }
  // acbp.py:_Reader: a field that does not fit reports the position it starts at
  auto need = [&](int64_t pos, int64_t len, const char* what) -> int {
    if (pos + len > nbytes) return ffail(pos, "truncated container: missing %s", what);
    return HLQ_OK;
  };
  HLQ_TRY(need(0, 4, "magic"));
  if (memcmp(h, "ACBP", 4) != 0) return ffail(0, "bad magic");
  HLQ_TRY(need(4, 2, "version"));
  const uint16_t version = uint16_t(h[4] | (h[5] << 8));
  if (version != 1) return ffail(4, "unsupported version %u", version);
  HLQ_TRY(need(6, 1, "bits"));
  const int bits = h[6];
  if (bits != 4 && bits != 8) return ffail(6, "unsupported bit width %d", bits);
  HLQ_TRY(need(7, 1, "block size"));
  const int block = h[7];
  if (block != 2 && block != 4 && block != 8 && block != 16) return ffail(7, "unsupported block size %d", block);
  HLQ_TRY(need(8, 2, "rank"));
  const int rank = h[8] | (h[9] << 8);
  if (rank < 1 || rank > block) return ffail(8, "rank %d out of range for block size %d", rank, block);
  HLQ_TRY(need(10, 2, "basis bitmap"));
  const uint32_t bitmap = uint32_t(h[10] | (h[11] << 8));
  if (bitmap >> block) return ffail(10, "basis bitmap 0x%04x has bits beyond the block", bitmap);
  if (__builtin_popcount(bitmap) != rank) return ffail(10, "basis bitmap 0x%04x does not select %d bases", bitmap, rank);
  HLQ_TRY(need(12, 1, "ndims"));
  if (h[12] != 3) return ffail(12, "unsupported ndims %d", int(h[12]));
  HLQ_TRY(need(13, 12, "dims"));
  uint32_t dims[3];
  memcpy(dims, h + 13, 12);
  HLQ_TRY(need(25, 4, "scale count"));
  uint32_t ns;
  memcpy(&ns, h + 25, 4);
  if (ns != 1) return ffail(25, "unsupported scale count %u", ns);
  HLQ_TRY(need(29, 4, "scale"));
  float scale;
  memcpy(&scale, h + 29, 4);
  if (!(scale > 0.0f) || scale == __builtin_inff()) return ffail(29, "scale must be positive and finite, got %g", double(scale));
  hlq_acbp_info inf{};
  inf.B = dims[0]; inf.L = dims[1]; inf.I = dims[2];
  inf.bits = bits; inf.block = block; inf.rank = rank; inf.bitmap = bitmap;
  container_geometry(inf.B, inf.L, inf.I, block, rank, &inf.axis, &inf.rows, &inf.K);
  const int64_t count = inf.rows * inf.K;
  inf.payload_bytes = bits == 8 ? count : (count + 1) / 2;
  inf.total_bytes = 33 + inf.payload_bytes + 4;
  if (nbytes != inf.total_bytes)
    return ffail(33, "container length %lld does not match the declared shape (expected %lld)", (long long)nbytes,
                 (long long)inf.total_bytes);
  *info = inf;
  return HLQ_OK;
}

int hlq_acbp_unpack(const uint8_t* buf, int64_t nbytes, const hlq_acbp_info* info, int8_t* payload, int64_t ld,
                    float* scale_out, void* ws, size_t ws_bytes, void* stream) {
  if (!info || nbytes != info->total_bytes) return fail(HLQ_ERR_PARAMETER, "info does not describe this buffer");
  if (ws_bytes < hlq_acbp_ws(nbytes)) return fail(HLQ_ERR_PARAMETER, "workspace too small");
  if (info->rows * info->K > 0 && (!payload || ld < info->K)) return fail(HLQ_ERR_DIMENSION, "payload ld < K");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t bad = -1;
  bool crc_ok = false;
  const int e = hlq::acbp_check_and_unpack(buf, nbytes, info->rows, info->K, info->bits, payload, ld, scale_out, ws,
                                           &bad, &crc_ok, st);
  if (e) return fail(HLQ_ERR_CUDA, "hlq_acbp_unpack: %s", cudaGetErrorString(cudaError_t(e)));
  if (bad >= 0)
    return ffail(33 + bad, info->bits == 8 ? "payload value out of the symmetric int8 range"
                                            : "payload value out of the symmetric int4 range");
  const int64_t count = info->rows * info->K;
  if (info->bits == 4 && (count % 2) && info->payload_bytes) {
    uint8_t last = 0;
    cudaMemcpy(&last, buf + 33 + info->payload_bytes - 1, 1, cudaMemcpyDeviceToHost);
    if (last >> 4) return ffail(33 + info->payload_bytes - 1, "nonzero padding nibble");
  }
  if (!crc_ok) return ffail(33 + info->payload_bytes, "crc mismatch");
  return HLQ_OK;
}

int hlq_conv_dgrad_i8_ex(const int8_t* gcodes, int64_t ld_g, int64_t B, int64_t Ho, int64_t Wo, int64_t O,
                         const int8_t* wcodes, int64_t ld_w, int64_t C, int k, int stride, int pad, int64_t H,
                         int64_t W, int bits, const float* sg, const float* sw, int epilogue, void* dx_nhwc,
                         int dx_dtype, int32_t* acc_out, void* stream) {
  HLQ_TRY(check_bits(bits));
  HLQ_TRY(check_dtype(dx_dtype));
  HLQ_TRY(check_ld16(ld_g, "gy codes"));
  HLQ_TRY(check_ld16(ld_w, "W codes"));
  if (B <= 0 || Ho <= 0 || Wo <= 0 || O <= 0 || C <= 0 || k <= 0 || stride <= 0 || stride > 8 || pad < 0 ||
      pad > k - 1 || ld_g < pad16(O) || ld_w < pad16(O) || k > 15 || H <= 0 || W <= 0 ||
      (H + 2 * pad - k) / stride + 1 != Ho || (W + 2 * pad - k) / stride + 1 != Wo || H + 2 * pad < k ||
      W + 2 * pad < k || B * H * W > INT32_MAX)
    return fail(HLQ_ERR_DIMENSION, "bad conv dgrad geometry");
  const long double worst = (long double)k * k * pad16(O) * qmax_of(bits) * qmax_of(bits);
  if (worst >= 2147483648.0L)
    return fail(HLQ_ERR_PARAMETER, "contraction k*k*O exceeds the int32-exact bound");
  if (epilogue != HLQ_EPI_EXACT && epilogue != HLQ_EPI_FAST)
    return fail(HLQ_ERR_PARAMETER, "unknown epilogue %d", epilogue);
  int e = hlq::launch_conv_dgrad_i8(gcodes, ld_g, B, Ho, Wo, O, wcodes, ld_w, C, k, stride, pad, H, W, sg, sw,
                                    epilogue, dx_nhwc, dx_dtype, C, acc_out, C, static_cast<cudaStream_t>(stream));
  if (e == -1) return fail(HLQ_ERR_CUDA, "im2col tensor map rejected");
  if (e != 0) return fail(HLQ_ERR_CUDA, "hlq_conv_dgrad_i8: %s", cudaGetErrorString(cudaError_t(e)));
  return HLQ_OK;
}

int hlq_conv_dgrad_i8(const int8_t* gcodes, int64_t ld_g, int64_t B, int64_t Ho, int64_t Wo, int64_t O,
                      const int8_t* wcodes, int64_t ld_w, int64_t C, int k, int stride, int pad,
                      int bits, const float* sg, const float* sw, int epilogue, void* dx_nhwc,
                      int dx_dtype, int32_t* acc_out, void* stream) {
  // stride 1 determines dX's extent; strided convs name it (hlq_conv_dgrad_i8_ex)
  if (stride != 1)
    return fail(HLQ_ERR_PARAMETER, "strided dgrad needs the dX extent: use hlq_conv_dgrad_i8_ex");
  return hlq_conv_dgrad_i8_ex(gcodes, ld_g, B, Ho, Wo, O, wcodes, ld_w, C, k, 1, pad, Ho + k - 1 - 2 * pad,
                              Wo + k - 1 - 2 * pad, bits, sg, sw, epilogue, dx_nhwc, dx_dtype, acc_out, stream);
}

int hlq_conv_acbp_compress(const void* x_nhwc, int dtype, int64_t B, int64_t H, int64_t W,
                           int64_t C, int k, int stride, int pad, uint32_t bitmap, int bits,
                           int8_t* payload, int64_t ld_payload, float* scale_out,
                           uint32_t* stats_ws, void* stream) {
  HLQ_TRY(check_dtype(dtype));
  HLQ_TRY(check_bits(bits));
  HLQ_TRY(check_bitmap(bitmap));
  HLQ_TRY(check_ld16(ld_payload, "payload"));
  if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || k <= 0 || stride <= 0 || pad < 0 ||
      H + 2 * pad < k || W + 2 * pad < k || B * H * W * C >= (int64_t(1) << 40))
    return fail(HLQ_ERR_DIMENSION, "bad conv geometry");
  const int64_t Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho * Wo < 16)
    return fail(HLQ_ERR_DIMENSION,
                "conv output has L=Ho*Wo=%lld < 16; the batch-axis projection needs the Python layer",
                (long long)(Ho * Wo));
  const int64_t kk = B * ((Ho * Wo + 15) / 16) * __builtin_popcount(bitmap);
  if (ld_payload < kk) return fail(HLQ_ERR_DIMENSION, "payload ld %lld < K %lld", (long long)ld_payload, (long long)kk);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool pooled = stats_ws == nullptr;  // library slot: the fused launch zeroes it again
  if (pooled) stats_ws = hlq::stats_slot();
  else cudaMemsetAsync(stats_ws, 0, HLQ_STATS_WS_BYTES, st);
  if (hlq::launch_conv_acbp_tma(x_nhwc, dtype, int(B), int(H), int(W), int(C), k, stride, pad, bitmap, bits,
                                hlq::kBoth, stats_ws, payload, ld_payload, scale_out, st, pooled))
    return cuda_status("hlq_conv_acbp_compress");
  if (pooled) cudaMemsetAsync(stats_ws, 0, HLQ_STATS_WS_BYTES, st);
  hlq::launch_im2col_proj(x_nhwc, dtype, int(B), int(H), int(W), int(C), k, stride, pad, bitmap, bits,
                          hlq::kStats, stats_ws, nullptr, 0, nullptr, st);
  hlq::launch_im2col_proj(x_nhwc, dtype, int(B), int(H), int(W), int(C), k, stride, pad, bitmap, bits,
                          hlq::kQuant, stats_ws, payload, ld_payload, scale_out, st);
  if (pooled) cudaMemsetAsync(stats_ws, 0, HLQ_STATS_WS_BYTES, st);  // leave the library slot zeroed
  return cuda_status("hlq_conv_acbp_compress");
}

int hlq_conv_acbp_pass(const void* x_nhwc, int dtype, int64_t B, int64_t H, int64_t W, int64_t C, int k,
                       int stride, int pad, uint32_t bitmap, int bits, int mode, uint32_t* stats_ws,
                       int8_t* payload, int64_t ld_payload, float* scale_out, void* stream) {
  HLQ_TRY(check_dtype(dtype));
  HLQ_TRY(check_bits(bits));
  HLQ_TRY(check_bitmap(bitmap));
  if (mode != 0 && mode != 1) return fail(HLQ_ERR_PARAMETER, "mode must be 0 (STATS) or 1 (QUANT)");
  if (mode == 1) HLQ_TRY(check_ld16(ld_payload, "payload"));
  if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || k <= 0 || stride <= 0 || pad < 0 ||
      H + 2 * pad < k || W + 2 * pad < k || B * H * W * C >= (int64_t(1) << 40))
    return fail(HLQ_ERR_DIMENSION, "bad conv geometry");
  const int64_t Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho * Wo < 16)
    return fail(HLQ_ERR_DIMENSION, "conv output has L=Ho*Wo=%lld < 16", (long long)(Ho * Wo));
  const int64_t kk = B * ((Ho * Wo + 15) / 16) * __builtin_popcount(bitmap);
  if (mode == 1 && ld_payload < kk)
    return fail(HLQ_ERR_DIMENSION, "payload ld %lld < K %lld", (long long)ld_payload, (long long)kk);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int m = mode == 0 ? hlq::kStats : hlq::kQuant;
  if (hlq::launch_conv_acbp_tma(x_nhwc, dtype, int(B), int(H), int(W), int(C), k, stride, pad, bitmap, bits, m,
                                stats_ws, payload, ld_payload, scale_out, st))
    return cuda_status("hlq_conv_acbp_pass");
  hlq::launch_im2col_proj(x_nhwc, dtype, int(B), int(H), int(W), int(C), k, stride, pad, bitmap, bits, m, stats_ws,
                          payload, ld_payload, scale_out, st);
  return cuda_status("hlq_conv_acbp_pass");
}

int hlq_col2im(const void* dcols, int dtype, int64_t ld, int64_t B, int64_t H, int64_t W, int64_t C,
               int k, int stride, int pad, void* dx_nhwc, int out_dtype, void* stream) {
  HLQ_TRY(check_dtype(dtype));
  HLQ_TRY(check_dtype(out_dtype));
  if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || k <= 0 || stride <= 0 || pad < 0 || ld < C * k * k)
    return fail(HLQ_ERR_DIMENSION, "bad col2im geometry");
  hlq::launch_col2im(dcols, dtype, ld, int(B), int(H), int(W), int(C), k, stride, pad, dx_nhwc,
                     out_dtype, static_cast<cudaStream_t>(stream));
  return cuda_status("hlq_col2im");
}

int hlq_col2im_ex(const void* dcols, int dtype, int64_t ld, int64_t B, int64_t H, int64_t W, int64_t C,
                  int k, int stride, int pad, int col_order, void* dx_nhwc, int out_dtype, void* stream) {
  if (col_order == 0)
    return hlq_col2im(dcols, dtype, ld, B, H, W, C, k, stride, pad, dx_nhwc, out_dtype, stream);
  if (col_order != 1) return fail(HLQ_ERR_PARAMETER, "col_order must be 0 (c, tap) or 1 (tap, c)");
  HLQ_TRY(check_dtype(dtype));
  HLQ_TRY(check_dtype(out_dtype));
  if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || k <= 0 || stride <= 0 || pad < 0 || ld < C * k * k)
    return fail(HLQ_ERR_DIMENSION, "bad col2im geometry");
  if (!hlq::launch_col2im_tapmajor(dcols, dtype, ld, int(B), int(H), int(W), int(C), k, stride, pad, dx_nhwc,
                                   out_dtype, static_cast<cudaStream_t>(stream)))
    return fail(HLQ_ERR_PARAMETER, "tap-major col2im needs C %% 8 == 0 and 16-byte aligned rows");
  return cuda_status("hlq_col2im_ex");
}

int64_t hlq_acbp_k(int64_t B, int64_t L, int axis, int rank) {
  return axis == 1 ? B * ((L + 15) / 16) * rank : ((B + 15) / 16) * rank;
}
int64_t hlq_acbp_rows(int64_t L, int64_t I, int axis) { return axis == 1 ? I : L * I; }

int hlq_acbp_compress(const void* x, int dtype, int64_t B, int64_t L, int64_t I, int axis,
                      uint32_t bitmap, int bits, int8_t* payload, int64_t ld_payload,
                      float* scale_out, uint32_t* stats_ws, void* stream) {
  if (axis != 0 && axis != 1) return fail(HLQ_ERR_PARAMETER, "axis must be 0 or 1, got %d", axis);
  // axis 1: B segments of (L x I); axis 0: one segment of (B x L*I) -- the
  // reference's (B_p r/16, L, I) payload flattens to rows (blk*r + j)*L + l,
  // which is exactly column (l*I + i) of the transposed projection.
  if (axis == 1)
    return hlq_quantize_proj_rows(x, dtype, B, L, I, I, L * I, bitmap, bits, stats_ws, payload,
                                  ld_payload, scale_out, stream);
  return hlq_quantize_proj_rows(x, dtype, 1, B, L * I, L * I, B * L * I, bitmap, bits, stats_ws,
                                payload, ld_payload, scale_out, stream);
}

size_t hlq_hq_grad_input_ws(int64_t T, int64_t O, int64_t I) {
  const int64_t op = pad16(O);
  return align256(size_t(T * op)) + align256(size_t(I * op)) + 2 * HLQ_STATS_WS_BYTES + 256;
}

int hlq_hq_grad_input(const void* gy, int gy_dtype, int64_t T, int64_t O, const float* w, int64_t I,
                      int bits, void* dx, int dx_dtype, int epilogue, void* ws, size_t ws_bytes,
                      void* stream) {
  HLQ_TRY(check_bits(bits));
  if (T < 0 || O <= 0 || I <= 0) return fail(HLQ_ERR_DIMENSION, "bad hq_grad_input shape");
  if (ws_bytes < hlq_hq_grad_input_ws(T, O, I))
    return fail(HLQ_ERR_PARAMETER, "workspace too small: %zu < %zu", ws_bytes,
                hlq_hq_grad_input_ws(T, O, I));
  const int64_t op = pad16(O);
  uint8_t* p = static_cast<uint8_t*>(ws);
  int8_t* cg = reinterpret_cast<int8_t*>(p);
  p += align256(size_t(T * op));
  int8_t* cw = reinterpret_cast<int8_t*>(p);
  p += align256(size_t(I * op));
  // one HLQ_STATS_WS_BYTES scratch per transform (statistics, grid barrier, work tickets)
  uint32_t* stats = reinterpret_cast<uint32_t*>(p);                             // gy
  uint32_t* stats_w = reinterpret_cast<uint32_t*>(p + HLQ_STATS_WS_BYTES);      // w
  float* scales = reinterpret_cast<float*>(p + 2 * HLQ_STATS_WS_BYTES);         // [0] gy, [1] w
  HLQ_TRY(hlq_quantize_ht_cols(gy, gy_dtype, T, O, O, bits, stats, cg, op, scales, stream));
  HLQ_TRY(hlq_quantize_proj_rows(w, HLQ_F32, 1, O, I, I, O * I, 0xFFFFu, bits, stats_w, cw, op,
                                 scales + 1, stream));
  return hlq_gemm_i8(cg, op, cw, op, T, I, op, bits, bits, scales, scales + 1, 1.0, epilogue, dx,
                     dx_dtype, I, nullptr, 0, stream);
}

size_t hlq_grad_weight_ws(int64_t B, int64_t L, int64_t O, int axis, int rank) {
  const int64_t k = hlq_acbp_k(B, L, axis, rank);
  return align256(size_t(hlq_acbp_rows(L, O, axis) * pad16(k))) + HLQ_STATS_WS_BYTES + 256;
}

size_t hlq_grad_weight_ws_ex(int64_t B, int64_t L, int64_t O, int64_t I, int axis, int rank, int bits) {
  // + the K-chunk slabs of a contraction past the int32-exact bound (hlq_gemm_i8_ws_bits)
  const int64_t k = hlq_acbp_k(B, L, axis, rank);
  return hlq_grad_weight_ws(B, L, O, axis, rank) + hlq_gemm_i8_ws_bits(O, I, k, axis == 0 ? L : 1, bits, bits);
}

int hlq_grad_weight(const int8_t* payload, int64_t ld_payload, const float* x_scale,
                    const void* gy, int gy_dtype, int64_t B, int64_t L, int64_t O, int64_t I,
                    int axis, uint32_t bitmap, int bits, double extra, void* dw, int dw_dtype,
                    int epilogue, void* ws, size_t ws_bytes, void* stream) {
  HLQ_TRY(check_bits(bits));
  HLQ_TRY(check_bitmap(bitmap));
  if (axis != 0 && axis != 1) return fail(HLQ_ERR_PARAMETER, "axis must be 0 or 1, got %d", axis);
  const int rank = __builtin_popcount(bitmap);
  const int64_t k = hlq_acbp_k(B, L, axis, rank);
  if (ld_payload < k)
    return fail(HLQ_ERR_STATE, "payload extent %lld < projected extent %lld", (long long)ld_payload,
                (long long)k);
  if (ws_bytes < hlq_grad_weight_ws(B, L, O, axis, rank))
    return fail(HLQ_ERR_PARAMETER, "workspace too small");
  const int64_t ldk = pad16(k);
  uint8_t* p = static_cast<uint8_t*>(ws);
  int8_t* cg = reinterpret_cast<int8_t*>(p);
  p += align256(size_t(hlq_acbp_rows(L, O, axis) * ldk));
  uint32_t* stats = reinterpret_cast<uint32_t*>(p);                      // HLQ_STATS_WS_BYTES
  float* scale = reinterpret_cast<float*>(p + HLQ_STATS_WS_BYTES);
  if (axis == 1)
    HLQ_TRY(hlq_quantize_proj_rows(gy, gy_dtype, B, L, O, O, L * O, bitmap, bits, stats, cg, ldk,
                                   scale, stream));
  else
    HLQ_TRY(hlq_quantize_proj_rows(gy, gy_dtype, 1, B, L * O, L * O, B * L * O, bitmap, bits, stats,
                                   cg, ldk, scale, stream));
  // axis 0: the transposed projections have L*O rows (l, o) and L*I rows
  // (l, i); the reference's K index (blk, j, l) becomes L stacked K panels.
  const int64_t groups = axis == 0 ? L : 1;
  // a workspace of hlq_grad_weight_ws_ex bytes also carries the GEMM's split / K-chunk slabs
  const size_t base = hlq_grad_weight_ws(B, L, O, axis, rank);
  void* gws = ws_bytes > base ? static_cast<uint8_t*>(ws) + base : nullptr;
  return hlq_gemm_i8_ex(cg, ldk, ldk * O, payload, ld_payload, ld_payload * I, O, I, k, groups, bits, bits, scale,
                        x_scale, extra, epilogue, dw, dw_dtype, I, nullptr, 0, gws, gws ? ws_bytes - base : 0,
                        stream);
}

}  // extern "C"
