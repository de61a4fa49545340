// True stochastic rounding on the GPU, bit-exact with the reference's
// quant_stochastic (quantize.py:114-125) and RngState (quantize.py:26-59):
//
//   up   = f64(q - floor(q)) > U,  q = RN(v / s) (fp32, IEEE division),
//   U    = the idx-th double of np.random.Generator(np.random.Philox(key=[seed, 0])).random(),
//   idx  = the element's C-order index in the array the reference quantizes,
//   seed = RngState(parent).split(tag).seed (splitmix64 on the host; tags
//          backprop.py:42-43 -- 11/12 the dX operands, 21/22 the dW operands).
//
// numpy's Philox is Philox4x64-10 (Random123): a 256-bit counter, 128-bit key;
// the generator increments the counter BEFORE each block, so raw uint64 #i is
// word (i mod 4) of block (i / 4 + 1), and random() = (raw >> 11) * 2^-53.
// Being counter-based, every element's draw is computed independently -- no
// stream state, any thread order.
//
// This is the QUANT pass only: the per-tensor scale comes from the regular
// STATS pass (the statistics do not depend on the rounding).  One thread per
// 16-vector: HT along the contiguous axis (gx operands) or the projection
// along rows (gw operands / ACBP / W codes), same butterfly as the fast
// kernels, same output layouts.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "hlq_internal.h"
#include "hlq_quant.cuh"
#include "hlq_philox.cuh"

namespace hlq {

namespace {

using namespace dev;

// quant_stochastic for one transformed value w (= 4 v, the unnormalised butterfly output)
__device__ __forceinline__ int quant_stoch(float w, float s, float qmax, double u) {
  const float v = __fmul_rn(w, 0.25f);
  const float q = __fdiv_rn(v, s);
  const float lo = floorf(q);
  const float frac = __fsub_rn(q, lo);
  float c = __fadd_rn(lo, double(frac) > u ? 1.0f : 0.0f);
  c = fminf(fmaxf(c, -qmax), qmax);
  return int(c);
}

struct SArgs {
  const void* src;
  int64_t segs, rows, cols, ld_src, seg_src, nblk;
  uint32_t bitmap;
  int rank, bits;
  const uint32_t* stats;  // {amax, ~minnz} of this operand
  int8_t* dst;
  int64_t ld_dst;
  float* scale_out;
  uint64_t k0, k1;  // Philox key [split seed, counter]
  int kind;         // gw index layout, see launch_stochastic_quant
  int64_t ktot, l2, o2;
};

template <typename T>
__device__ __forceinline__ float ld_src(const SArgs& a, int64_t s, int64_t r, int64_t c) {
  if (r >= a.rows || c >= a.cols) return 0.0f;
  const T* p = static_cast<const T*>(a.src) + s * a.seg_src + r * a.ld_src + c;
  if (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  return *reinterpret_cast<const float*>(p);
}

__device__ __forceinline__ float scale_of(const SArgs& a) {
  const Quant q = make_quant(a.stats, a.bits);
  return q.s;
}

// gx operands: 16-point HT along the contiguous axis; unit = (segment row t, block b)
template <typename T>
__global__ void __launch_bounds__(256) stoch_cols_kernel(SArgs a) {
  const float s = scale_of(a);
  const float qmax = float((1 << (a.bits - 1)) - 1);
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.scale_out) *a.scale_out = s;
  const int64_t nb = (a.cols + 15) / 16, ldi = nb * 16, units = a.segs * a.rows * nb;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = u / nb, b = u - t * nb;
    const int64_t sg = t / a.rows, r = t - sg * a.rows;
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = ld_src<T>(a, sg, r, b * 16 + j);
    fwht16_raw(v);
    const uint64_t idx0 = uint64_t(t * ldi + b * 16);
    uint32_t packed[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      double uu[4];
      philox_u01_x4(a.k0, a.k1, idx0 + 4 * g, uu);
      uint32_t p = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) p |= (uint32_t(quant_stoch(v[4 * g + i], s, qmax, uu[i])) & 0xFFu) << (8 * i);
      packed[g] = p;
    }
    *reinterpret_cast<uint4*>(a.dst + t * a.ld_dst + b * 16) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
}

// gw operands / ACBP / W codes: projection along rows; unit = (column c, global block gb)
template <typename T>
__global__ void __launch_bounds__(256) stoch_rows_kernel(SArgs a) {
  const float s = scale_of(a);
  const float qmax = float((1 << (a.bits - 1)) - 1);
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.scale_out) *a.scale_out = s;
  const int64_t units = a.cols * a.segs * a.nblk;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t gb = u / a.cols, c = u - gb * a.cols;  // consecutive threads: consecutive columns
    const int64_t sg = gb / a.nblk, blk = gb - sg * a.nblk;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = ld_src<T>(a, sg, blk * 16 + i, c);
    fwht16_raw(v);
    int j = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!((a.bitmap >> i) & 1u)) continue;
      const int64_t k = gb * a.rank + j;
      uint64_t idx;
      if (a.kind == 0) idx = uint64_t(c * a.ktot + k);                 // (cols, K): gy gw-left, transposed
      else if (a.kind == 1) idx = uint64_t(k * a.cols + c);            // (K, cols): ACBP of x, W codes
      else {                                                           // batch axis, L > 1: c = l*O + o
        const int64_t o = c % a.o2, l = c / a.o2;
        idx = uint64_t(o * (a.ktot * a.l2) + k * a.l2 + l);
      }
      a.dst[c * a.ld_dst + k] = int8_t(quant_stoch(v[i], s, qmax, philox_u01(a.k0, a.k1, idx)));
      ++j;
    }
  }
}

}  // namespace

void launch_stochastic_quant(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols, int64_t ld_src,
                             int64_t seg_src, bool along_cols, uint32_t bitmap, int bits, const uint32_t* stats,
                             int8_t* dst, int64_t ld_dst, float* scale_out, uint64_t k0, uint64_t k1, int kind,
                             int64_t l2, int64_t o2, cudaStream_t st) {
  SArgs a{};
  a.src = src; a.segs = segs; a.rows = rows; a.cols = cols; a.ld_src = ld_src; a.seg_src = seg_src;
  a.nblk = (rows + 15) / 16; a.bitmap = bitmap; a.rank = __builtin_popcount(bitmap); a.bits = bits;
  a.stats = stats; a.dst = dst; a.ld_dst = ld_dst; a.scale_out = scale_out; a.k0 = k0; a.k1 = k1;
  a.kind = kind; a.ktot = segs * a.nblk * a.rank; a.l2 = l2; a.o2 = o2;
  const int64_t units = along_cols ? segs * rows * ((cols + 15) / 16) : cols * segs * a.nblk;
  int64_t grid = (units + 255) / 256;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  if (grid < 1) grid = 1;
  if (along_cols) {
    if (dtype == kBF16) stoch_cols_kernel<__nv_bfloat16><<<int(grid), 256, 0, st>>>(a);
    else stoch_cols_kernel<float><<<int(grid), 256, 0, st>>>(a);
  } else {
    if (dtype == kBF16) stoch_rows_kernel<__nv_bfloat16><<<int(grid), 256, 0, st>>>(a);
    else stoch_rows_kernel<float><<<int(grid), 256, 0, st>>>(a);
  }
}

}  // namespace hlq

// ---------------------------------------------------------------------------
// Basis energy for calibrated basis selection (train.py:128-134 _basis_energy,
// hadamard.py:174-188 select_bases): sum over every 16-row block and column of
// |coefficient i| of the orthonormal block transform along rows, i = 0..15,
// accumulated in fp64 (the ordering of the per-basis means is what selection
// uses).  energy (16 doubles) is zeroed by the caller's stream first.
// ---------------------------------------------------------------------------
namespace hlq {
namespace {

template <typename T>
__global__ void __launch_bounds__(256) basis_energy_kernel(const void* src, int64_t segs, int64_t rows, int64_t cols,
                                                           int64_t ld_src, int64_t seg_src, double* energy) {
  const int64_t nblk = (rows + 15) / 16, units = cols * segs * nblk;
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t gb = u / cols, c = u - gb * cols;
    const int64_t sg = gb / nblk, blk = gb - sg * nblk;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t r = blk * 16 + i;
      float x = 0.0f;
      if (r < rows) {
        const T* p = static_cast<const T*>(src) + sg * seg_src + r * ld_src + c;
        x = sizeof(T) == 2 ? __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p))
                           : *reinterpret_cast<const float*>(p);
      }
      v[i] = x;
    }
    dev::fwht16_raw(v);
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] += double(fabsf(__fmul_rn(v[i], 0.25f)));
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double a = acc[i];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(energy + i, a);
  }
}

}  // namespace

void launch_basis_energy(const void* src, int dtype, int64_t segs, int64_t rows, int64_t cols, int64_t ld_src,
                         int64_t seg_src, double* energy, cudaStream_t st) {
  cudaMemsetAsync(energy, 0, 16 * sizeof(double), st);
  const int64_t units = cols * segs * ((rows + 15) / 16);
  int64_t grid = (units + 255) / 256;
  if (grid > num_sms() * 8) grid = num_sms() * 8;
  if (grid < 1) grid = 1;
  if (dtype == kBF16)
    basis_energy_kernel<__nv_bfloat16><<<int(grid), 256, 0, st>>>(src, segs, rows, cols, ld_src, seg_src, energy);
  else
    basis_energy_kernel<float><<<int(grid), 256, 0, st>>>(src, segs, rows, cols, ld_src, seg_src, energy);
}

}  // namespace hlq
