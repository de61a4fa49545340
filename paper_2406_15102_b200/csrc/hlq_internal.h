// Internal launch declarations shared by the kernel translation units and the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace hlq {

enum : int { kF32 = 0, kBF16 = 1 };
enum : int { kStats = 0, kQuant = 1 };
enum : int { kEpiExact = 0, kEpiFast = 1 };

int num_sms();

void launch_ht_cols_any(const void* src, int dtype, int64_t rows, int64_t cols, int64_t ld_src,
                        int bits, int mode, uint32_t* amax_bits, int8_t* dst, int64_t ld_dst,
                        float* scale_out, cudaStream_t stream);

void launch_proj_rows_any(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                          int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits, int mode,
                          uint32_t* amax_bits, int8_t* dst, int64_t ld_dst, float* scale_out,
                          cudaStream_t stream);

// Returns a cudaError_t-compatible code (0 on success) or -1 if the tensor maps
// could not be encoded.
int launch_gemm_i8(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int64_t M, int64_t N,
                   int64_t K, int64_t groups, int64_t a_gstride, int64_t b_gstride,
                   const float* sa, const float* sb, double extra, int epilogue,
                   void* out, int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc,
                   cudaStream_t stream);

}  // namespace hlq
