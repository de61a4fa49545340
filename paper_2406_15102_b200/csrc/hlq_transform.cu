// Block-Hadamard transform + per-tensor amax + pseudo-stochastic quantizer.
//
// Two kernel families cover every operand of the HLQ backward:
//
//  * ht_cols  -- 16-point FWHT along the CONTIGUOUS axis of a (T, C) matrix,
//                full rank, codes written row-major (T, C_pad16).  This is the
//                gx left operand Q(H.gy) (backprop.py:362,367).
//  * proj_rows -- 16-point FWHT along the ROW axis of S segments of (R, C),
//                keeping the `rank` bases selected by a 16-bit bitmap, codes
//                written TRANSPOSED as (C, K) with K = S * ceil(R/16) * rank, so
//                the result is directly a K-major tcgen05 operand.  Used for the
//                gw operands P.gy and P.X (ACBP, backprop.py:223-234,373-410)
//                and, at rank 16, for the gx right operand H.W (backprop.py:363).
//
// Each family has a STATS pass (max |v| over the transformed tensor, reduced
// with one atomicMax on the IEEE bits per CTA -- |v| >= 0 so the unsigned
// order is the float order, and any NaN/Inf lands above 0x7F800000, which is
// how non-finite input is reported) and a QUANT pass (recompute the
// transform, scale = amax / qmax, pseudo-stochastic rounding).
//
// Bit-exactness contract: butterfly stages in the order
// h = 1, 2, 4, 8 with (lower, upper) = (a + b, a - b); one multiply by 0.25;
// IEEE division v / scale (div.rn, never v * rcp); no FTZ.  The explicit
// __f*_rn intrinsics keep nvcc from contracting or reassociating anything.
#include <cuda_bf16.h>
#include <cstdint>

#include "hlq_internal.h"
#include "hlq_ptx.cuh"

namespace hlq {

namespace {

// Load 4 consecutive elements; vector path when the caller proved alignment.
template <typename T>
__device__ __forceinline__ void load4(const T* p, int64_t valid, bool vec, float (&o)[4]);

template <>
__device__ __forceinline__ void load4<float>(const float* p, int64_t valid, bool vec, float (&o)[4]) {
  if (vec && valid >= 4) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = j < valid ? __ldg(p + j) : 0.0f;
  }
}

template <>
__device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16* p, int64_t valid, bool vec,
                                                     float (&o)[4]) {
  if (vec && valid >= 4) {
    uint2 raw = __ldg(reinterpret_cast<const uint2*>(p));
    o[0] = __uint_as_float(raw.x << 16);
    o[1] = __uint_as_float(raw.x & 0xFFFF0000u);
    o[2] = __uint_as_float(raw.y << 16);
    o[3] = __uint_as_float(raw.y & 0xFFFF0000u);
  } else {
    const unsigned short* q = reinterpret_cast<const unsigned short*>(p);
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = j < valid ? __uint_as_float(uint32_t(__ldg(q + j)) << 16) : 0.0f;
  }
}

// Orthonormal 16-point FWHT in registers (hadamard.py:121-134 stage order).
__device__ __forceinline__ void fwht16(float (&v)[16]) {
#pragma unroll
  for (int h = 1; h < 16; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!(i & h)) {
        const float a = v[i], b = v[i + h];
        v[i] = __fadd_rn(a, b);
        v[i + h] = __fsub_rn(a, b);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __fmul_rn(v[i], 0.25f);
}

__device__ __forceinline__ uint32_t abs_bits(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

// scale = f32(amax) / f32(qmax); 0 -> 1  (quantize.py:94-100)
__device__ __forceinline__ float scale_from_amax(uint32_t amax_bits, float qmax) {
  const float s = __fdiv_rn(__uint_as_float(amax_bits), qmax);
  return s == 0.0f ? 1.0f : s;
}

// quantize.py:128-145 for one value.
__device__ __forceinline__ int quant_code(float v, float scale, float qmax) {
  const float q = __fdiv_rn(v, scale);
  const float lo = floorf(q);
  const float draw = __uint2float_rn(__float_as_uint(v) & 0x7FFu);
  const float frac = __fmul_rn(__fsub_rn(q, lo), 2048.0f);
  float c = __fadd_rn(lo, frac > draw ? 1.0f : 0.0f);
  c = fminf(fmaxf(c, -qmax), qmax);
  return static_cast<int>(c);
}

__device__ __forceinline__ void block_reduce_max_atomic(uint32_t v, uint32_t* amax_bits) {
  __shared__ uint32_t red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = l < nw ? red[l] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0 && v != 0u) atomicMax(amax_bits, v);
  }
}

// ---------------------------------------------------------------------------
// ht_cols: FWHT along the contiguous axis, 4 columns per thread, 4 threads
// per 16-block (stages h=1,2 in-thread, h=4,8 via lane shuffles).
// ---------------------------------------------------------------------------
template <typename T, int MODE>
__global__ void __launch_bounds__(256) ht_cols_kernel(const T* __restrict__ src, int64_t rows,
                                                       int64_t cols, int64_t ld_src, bool vec,
                                                       float qmax, uint32_t* __restrict__ amax_bits,
                                                       int8_t* __restrict__ dst, int64_t ld_dst,
                                                       float* __restrict__ scale_out) {
  const int64_t cols_p = (cols + 15) & ~int64_t(15);
  const int64_t groups = cols_p >> 2;  // multiple of 4: a 16-block never straddles lanes 4k..4k+3
  const int64_t total = rows * groups;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  float scale = 1.0f;
  if (MODE == kQuant) {
    scale = scale_from_amax(*amax_bits, qmax);
    if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
  }
  const int sub = threadIdx.x & 3;
  uint32_t lmax = 0;
  // total is rounded so every lane of a warp iterates the same number of times;
  // (r, g) advance incrementally so the loop carries no 64-bit division.
  const int64_t total_r = (total + stride - 1) / stride * stride;
  const int64_t step_r = stride / groups, step_g = stride - step_r * groups;
  int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t r = it / groups, g = it - r * groups;
  for (; it < total_r; it += stride) {
    const bool live = it < total;
    const int64_t c0 = g << 2;
    float x[4];
    load4<T>(src + (live ? r * ld_src + c0 : 0), live ? cols - c0 : 0, vec, x);
    // h = 1, 2 inside the thread
    {
      float a = x[0], b = x[1];
      x[0] = __fadd_rn(a, b); x[1] = __fsub_rn(a, b);
      a = x[2]; b = x[3];
      x[2] = __fadd_rn(a, b); x[3] = __fsub_rn(a, b);
      a = x[0]; b = x[2];
      x[0] = __fadd_rn(a, b); x[2] = __fsub_rn(a, b);
      a = x[1]; b = x[3];
      x[1] = __fadd_rn(a, b); x[3] = __fsub_rn(a, b);
    }
    // h = 4 (partner lane ^ 1), h = 8 (partner lane ^ 2): lower = a + b, upper = a - b
#pragma unroll
    for (int m = 1; m <= 2; m <<= 1) {
      const bool upper = sub & m;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float other = __shfl_xor_sync(0xffffffffu, x[k], m);
        x[k] = upper ? __fsub_rn(other, x[k]) : __fadd_rn(x[k], other);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __fmul_rn(x[k], 0.25f);
    const int64_t r_cur = r;
    r += step_r;
    g += step_g;
    if (g >= groups) { g -= groups; ++r; }
    if (!live) continue;
    if (MODE == kStats) {
#pragma unroll
      for (int k = 0; k < 4; ++k) lmax = max(lmax, abs_bits(x[k]));
    } else {
      uint32_t packed = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        packed |= (uint32_t(quant_code(x[k], scale, qmax)) & 0xFFu) << (8 * k);
      *reinterpret_cast<uint32_t*>(dst + r_cur * ld_dst + c0) = packed;
    }
  }
  if (MODE == kStats) block_reduce_max_atomic(lmax, amax_bits);
}

// ---------------------------------------------------------------------------
// proj_rows: FWHT along rows in 16-row blocks inside each segment, keep the
// bitmap's bases, write codes transposed: dst[c * ld_dst + gb * rank + j]
// where gb = s * nblk + blk is the global block index.  One thread = one
// 16-row block x 4 columns (64 fp32 values in registers).
// ---------------------------------------------------------------------------
template <typename T, int MODE>
__global__ void __launch_bounds__(256) proj_rows_kernel(
    const T* __restrict__ src, int64_t segs, int64_t rows, int64_t cols, int64_t ld_src,
    int64_t seg_src, bool vec, uint32_t bitmap, int rank, float qmax,
    uint32_t* __restrict__ amax_bits, int8_t* __restrict__ dst, int64_t ld_dst,
    float* __restrict__ scale_out) {
  const int64_t nblk = (rows + 15) >> 4;
  const int64_t groups = (cols + 3) >> 2;
  const int64_t total = segs * nblk * groups;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  float scale = 1.0f;
  if (MODE == kQuant) {
    scale = scale_from_amax(*amax_bits, qmax);
    if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
  }
  uint32_t lmax = 0;
  for (int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; it < total; it += stride) {
    const int64_t gb = it / groups;
    const int64_t g = it - gb * groups;
    const int64_t s = gb / nblk;
    const int64_t blk = gb - s * nblk;
    const int64_t c0 = g << 2;
    const int64_t cvalid = cols - c0;
    const int64_t rvalid = rows - (blk << 4);
    const T* base = src + s * seg_src + (blk << 4) * ld_src + c0;
    float v[4][16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float t[4];
      load4<T>(base + i * ld_src, i < rvalid ? cvalid : 0, vec, t);
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k][i] = t[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) fwht16(v[k]);
    if (MODE == kStats) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int b = 0; b < 16; ++b)
          if ((bitmap >> b) & 1u) lmax = max(lmax, abs_bits(v[k][b]));
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k >= cvalid) break;
        uint64_t lo = 0, hi = 0;
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          if ((bitmap >> b) & 1u) {
            const int j = __popc(bitmap & ((1u << b) - 1u));
            const uint64_t code = uint64_t(uint32_t(quant_code(v[k][b], scale, qmax)) & 0xFFu);
            if (j < 8) lo |= code << (8 * j); else hi |= code << (8 * (j - 8));
          }
        }
        int8_t* out = dst + (c0 + k) * ld_dst + gb * rank;
        // rank in {2,4,8,16} with ld_dst % 16 == 0 keeps these stores naturally aligned
        if (rank == 16) {
          *reinterpret_cast<uint4*>(out) = make_uint4(uint32_t(lo), uint32_t(lo >> 32), uint32_t(hi),
                                                      uint32_t(hi >> 32));
        } else if (rank == 8) {
          *reinterpret_cast<uint64_t*>(out) = lo;
        } else if (rank == 4) {
          *reinterpret_cast<uint32_t*>(out) = uint32_t(lo);
        } else if (rank == 2) {
          *reinterpret_cast<uint16_t*>(out) = uint16_t(lo);
        } else {
          for (int j = 0; j < rank; ++j)
            out[j] = int8_t(j < 8 ? (lo >> (8 * j)) & 0xFF : (hi >> (8 * (j - 8))) & 0xFF);
        }
      }
    }
  }
  if (MODE == kStats) block_reduce_max_atomic(lmax, amax_bits);
}

int grid_for(int64_t items, int threads) {
  const int64_t want = (items + threads - 1) / threads;
  const int64_t cap = int64_t(num_sms()) * 8;
  return int(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

template <typename T>
static void launch_ht_cols(const void* src, int64_t rows, int64_t cols, int64_t ld_src, int bits,
                           int mode, uint32_t* amax_bits, int8_t* dst, int64_t ld_dst,
                           float* scale_out, cudaStream_t stream) {
  const float qmax = float((1 << (bits - 1)) - 1);
  const bool vec = (reinterpret_cast<uintptr_t>(src) % (4 * sizeof(T)) == 0) && (ld_src % 4 == 0);
  const int64_t items = rows * (((cols + 15) & ~int64_t(15)) >> 2);
  const int threads = 256;
  const int grid = grid_for(items, threads);
  const T* s = static_cast<const T*>(src);
  if (mode == kStats)
    ht_cols_kernel<T, kStats><<<grid, threads, 0, stream>>>(s, rows, cols, ld_src, vec, qmax,
                                                             amax_bits, dst, ld_dst, scale_out);
  else
    ht_cols_kernel<T, kQuant><<<grid, threads, 0, stream>>>(s, rows, cols, ld_src, vec, qmax,
                                                             amax_bits, dst, ld_dst, scale_out);
}

template <typename T>
static void launch_proj_rows(const void* src, int64_t segs, int64_t rows, int64_t cols,
                             int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits, int mode,
                             uint32_t* amax_bits, int8_t* dst, int64_t ld_dst, float* scale_out,
                             cudaStream_t stream) {
  const float qmax = float((1 << (bits - 1)) - 1);
  const bool vec = (reinterpret_cast<uintptr_t>(src) % (4 * sizeof(T)) == 0) && (ld_src % 4 == 0) &&
                   (seg_src % 4 == 0);
  const int rank = __builtin_popcount(bitmap);
  const int64_t items = segs * ((rows + 15) >> 4) * ((cols + 3) >> 2);
  const int threads = 256;
  const int grid = grid_for(items, threads);
  const T* s = static_cast<const T*>(src);
  if (mode == kStats)
    proj_rows_kernel<T, kStats><<<grid, threads, 0, stream>>>(
        s, segs, rows, cols, ld_src, seg_src, vec, bitmap, rank, qmax, amax_bits, dst, ld_dst,
        scale_out);
  else
    proj_rows_kernel<T, kQuant><<<grid, threads, 0, stream>>>(
        s, segs, rows, cols, ld_src, seg_src, vec, bitmap, rank, qmax, amax_bits, dst, ld_dst,
        scale_out);
}

void launch_ht_cols_any(const void* src, int dtype, int64_t rows, int64_t cols, int64_t ld_src,
                        int bits, int mode, uint32_t* amax_bits, int8_t* dst, int64_t ld_dst,
                        float* scale_out, cudaStream_t stream) {
  if (dtype == kBF16)
    launch_ht_cols<__nv_bfloat16>(src, rows, cols, ld_src, bits, mode, amax_bits, dst, ld_dst,
                                  scale_out, stream);
  else
    launch_ht_cols<float>(src, rows, cols, ld_src, bits, mode, amax_bits, dst, ld_dst, scale_out,
                          stream);
}

void launch_proj_rows_any(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols,
                          int64_t ld_src, int64_t seg_src, uint32_t bitmap, int bits, int mode,
                          uint32_t* amax_bits, int8_t* dst, int64_t ld_dst, float* scale_out,
                          cudaStream_t stream) {
  if (dtype == kBF16)
    launch_proj_rows<__nv_bfloat16>(src, segs, rows, cols, ld_src, seg_src, bitmap, bits, mode,
                                    amax_bits, dst, ld_dst, scale_out, stream);
  else
    launch_proj_rows<float>(src, segs, rows, cols, ld_src, seg_src, bitmap, bits, mode, amax_bits,
                            dst, ld_dst, scale_out, stream);
}

}  // namespace hlq
