// Kernels for the reference's baseline gradient paths:
// the ablation strategies of backprop.py:91-155 that are not HLQ --
//   quant     naive int4/int8: quantize gy / W / x directly (backprop.py:272-279, 301-307)
//   ht_quant  on dW: full-rank block transform along the token axis (backprop.py:256-269)
//   lowrank   LBP-WHT: float projection, float GEMM, inverse projection of dX
//             (backprop.py:212-249, 310-316)
//   bits=None float pipelines (float_pipeline / debug_exact, backprop.py:120-137)
//
// One strided "view" drives every kernel: unit (segment s, 16-block b along
// the transform axis, column c), source element (s, r, c) at
// s*ss + r*sr + c*sc.  The transform is the block FWHT along r with the bases
// of `bitmap` kept (0xFFFF: _block_axis; 0: identity, no transform, r indexes
// the output directly).  Output (s, k, c) goes to s*ds + k*dk + c*dc, with
// k = b*rank + j for the j-th kept basis, and its C-order index in the array
// the reference quantizes is s*is + k*ik + c*ic (the Philox draw index).
// Consecutive threads take consecutive columns, so views with sc == 1 read
// coalesced.  These are accuracy-study paths: plain one-pass-per-stage
// kernels, not tuned like the HLQ hot path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "hlq_internal.h"
#include "hlq_philox.cuh"
#include "hlq_quant.cuh"

namespace hlq {

namespace {

using namespace dev;

template <typename T>
__device__ __forceinline__ float load_el(const XformView& x, int64_t s, int64_t r, int64_t c) {
  const T* p = static_cast<const T*>(x.src) + s * x.ss + r * x.sr + c * x.sc;
  if (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  return *reinterpret_cast<const float*>(p);
}

// The 16 outputs of unit (s, b, c): normalised coefficients (transform) or the
// raw values (identity).  Returns the number of valid outputs (identity: rows
// left in the block; transform: 16, the caller applies the bitmap).
template <typename T>
__device__ __forceinline__ int unit_values(const XformView& x, int64_t s, int64_t b, int64_t c, float (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int64_t r = b * 16 + i;
    v[i] = r < x.rows ? load_el<T>(x, s, r, c) : 0.0f;
  }
  if (x.bitmap == 0) {
    const int64_t left = x.rows - b * 16;
    return left < 16 ? int(left) : 16;
  }
  fwht16_raw(v);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __fmul_rn(v[i], 0.25f);  // orthonormal (exact power of two)
  return 16;
}

template <typename F>
__device__ __forceinline__ void for_each_output(const XformView& x, const float (&v)[16], int n, int64_t b, F&& f) {
  if (x.bitmap == 0) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < n) f(b * 16 + i, v[i]);
    return;
  }
  int j = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (!((x.bitmap >> i) & 1u)) continue;
    f(b * x.rank + j, v[i]);
    ++j;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) xform_stats_kernel(XformView x, uint32_t* stats) {
  Stat st;
  const int64_t units = x.segs * x.nblk * x.cols;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t sb = u / x.cols, c = u - sb * x.cols;
    const int64_t s = sb / x.nblk, b = sb - s * x.nblk;
    float v[16];
    const int n = unit_values<T>(x, s, b, c, v);
    for_each_output(x, v, n, b, [&](int64_t, float val) { st.add(val); });
  }
  st.warp_reduce();
  if ((threadIdx.x & 31) == 0) st.commit(stats);
}

// scale = f32(amax) / f32(qmax), 0 -> 1 (quantize.py:94-100)
__device__ __forceinline__ float scale_from(const uint32_t* stats, float qmax) {
  const float amax = __uint_as_float(__ldcg(stats));
  const float s = __fdiv_rn(amax, qmax);
  return s == 0.0f ? 1.0f : s;
}

template <typename T>
__global__ void __launch_bounds__(256) xform_quant_kernel(XformView x, int bits, int rounding, uint64_t k0,
                                                          uint64_t k1, const uint32_t* stats, int8_t* dst,
                                                          float* scale_out) {
  const float qmax = float((1 << (bits - 1)) - 1);
  const float sc = scale_from(stats, qmax);
  if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = sc;
  const int64_t units = x.segs * x.nblk * x.cols;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t sb = u / x.cols, c = u - sb * x.cols;
    const int64_t s = sb / x.nblk, b = sb - s * x.nblk;
    float v[16];
    const int n = unit_values<T>(x, s, b, c, v);
    for_each_output(x, v, n, b, [&](int64_t k, float val) {
      const float q = __fdiv_rn(val, sc);
      const float lo = floorf(q);
      const float frac = __fsub_rn(q, lo);
      bool up;
      if (rounding == 0) {  // quant_pseudo_stochastic (quantize.py:128-145)
        up = __fmul_rn(frac, 2048.0f) > __uint2float_rn(__float_as_uint(val) & 0x7FFu);
      } else {              // quant_stochastic (quantize.py:114-125)
        const uint64_t idx = uint64_t(s * x.is + k * x.ik + c * x.ic);
        up = double(frac) > philox_u01(k0, k1, idx);
      }
      const float code = fminf(fmaxf(__fadd_rn(lo, up ? 1.0f : 0.0f), -qmax), qmax);
      dst[s * x.ds + k * x.dk + c * x.dc] = int8_t(int(code));
    });
  }
}

template <typename T>
__global__ void __launch_bounds__(256) xform_f32_kernel(XformView x, float* dst) {
  const int64_t units = x.segs * x.nblk * x.cols;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t sb = u / x.cols, c = u - sb * x.cols;
    const int64_t s = sb / x.nblk, b = sb - s * x.nblk;
    float v[16];
    const int n = unit_values<T>(x, s, b, c, v);
    for_each_output(x, v, n, b, [&](int64_t k, float val) { dst[s * x.ds + k * x.dk + c * x.dc] = val; });
  }
}

// _unproject_axis (backprop.py:237-249): scatter the kept coefficients of a
// block into 16 slots (zeros elsewhere), orthonormal FWHT, crop to `rows`.
// Here the view's SOURCE strides index the coefficients (s, k, c) and the
// DESTINATION strides the output (s, r, c).
__global__ void __launch_bounds__(256) unproject_kernel(XformView x, float* dst) {
  const int64_t units = x.segs * x.nblk * x.cols;
  const float* src = static_cast<const float*>(x.src);
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t sb = u / x.cols, c = u - sb * x.cols;
    const int64_t s = sb / x.nblk, b = sb - s * x.nblk;
    float v[16];
    int j = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = 0.0f;
      if ((x.bitmap >> i) & 1u) {
        v[i] = src[s * x.ss + (b * x.rank + j) * x.sr + c * x.sc];
        ++j;
      }
    }
    fwht16_raw(v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t r = b * 16 + i;
      if (r < x.rows) dst[s * x.ds + r * x.dk + c * x.dc] = __fmul_rn(v[i], 0.25f);
    }
  }
}

int grid_for(const XformView& x) {
  const int64_t units = x.segs * x.nblk * x.cols;
  int64_t g = (units + 255) / 256;
  if (g > num_sms() * 16) g = num_sms() * 16;
  return int(g < 1 ? 1 : g);
}

}  // namespace

void launch_xform_quant(const XformView& x, int bits, int rounding, uint64_t k0, uint64_t k1, uint32_t* stats,
                        int8_t* dst, float* scale_out, cudaStream_t st) {
  cudaMemsetAsync(stats, 0, 2 * sizeof(uint32_t), st);
  const int g = grid_for(x);
  if (x.dtype == kBF16) {
    xform_stats_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(x, stats);
    xform_quant_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(x, bits, rounding, k0, k1, stats, dst, scale_out);
  } else {
    xform_stats_kernel<float><<<g, 256, 0, st>>>(x, stats);
    xform_quant_kernel<float><<<g, 256, 0, st>>>(x, bits, rounding, k0, k1, stats, dst, scale_out);
  }
}

void launch_xform_f32(const XformView& x, float* dst, cudaStream_t st) {
  const int g = grid_for(x);
  if (x.dtype == kBF16) xform_f32_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(x, dst);
  else xform_f32_kernel<float><<<g, 256, 0, st>>>(x, dst);
}

void launch_unproject_f32(const XformView& x, float* dst, cudaStream_t st) {
  unproject_kernel<<<grid_for(x), 256, 0, st>>>(x, dst);
}

}  // namespace hlq
