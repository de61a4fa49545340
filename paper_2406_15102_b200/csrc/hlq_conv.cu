// Conv2d lowering kernels for the HLQ path (harness/layers.py:96-158).
//
// The reference lowers a k x k convolution to a GEMM with
//   cols[b, l, c*k*k + i*k + j] = x[b, c, ho*s - p + i, wo*s - p + j]   (0 outside)
//   l = ho*Wo + wo,  L = Ho*Wo,  I = C*k*k
// and runs the Linear HLQ path on (cols, W.reshape(O, I), gy (B, L, O)).
//
//  * im2col_proj: ACBP of cols WITHOUT materialising cols: for each tap (i, j)
//    and 256-channel tile, 16-output-pixel blocks are gathered straight from
//    channels-last x (16 consecutive channels = one 32/64-byte load), FWHT'd
//    along the pixel axis, reduced to the plan's bases and quantized; codes go
//    to row c*k*k + i*k + j of the K-major payload, K = B * ceil(L/16) * r.
//    Same quantizer as the transform kernels (bit-exact vs acbp_compress).
//  * col2im: dX[b, h, w, c] = sum over taps (i, j) in the reference's (i, j)
//    order of dcols[b*L + l(h, w, i, j), c*k*k + i*k + j]; fp32 accumulation
//    in that order reproduces the reference's np scatter-add bit for bit.
#include <cuda_bf16.h>
#include <cstdint>

#include "hlq_internal.h"
#include "hlq_ptx.cuh"
#include "hlq_quant.cuh"

namespace hlq {

namespace {

using namespace dev;

constexpr int kCols = 256;
constexpr int kThreads = 256;

struct ConvArgs {
  const void* x;  // channels-last (B, H, W, C)
  int B, H, W, C, k, stride, pad, Ho, Wo, L, nblk, rank, bits;
  uint32_t bitmap;
  int nb, ctiles, items;
  uint32_t* stats;  // {amax, ~minnz} at [2..3] (gw slot)
  int8_t* dst;
  int64_t ld_dst;
  float* scale;
  uint32_t* nonfinite;  // nonfinite_word()
  bool vec;
};

template <typename T>
__device__ __forceinline__ void load16(const T* p, int n, bool vec, float (&v)[16]) {
  if (sizeof(T) == 2) {
    const unsigned short* q = reinterpret_cast<const unsigned short*>(p);
    if (vec && n == 16) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(p) + h);
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) { v[8 * h + 2 * k] = bf_lo(w[k]); v[8 * h + 2 * k + 1] = bf_hi(w[k]); }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = i < n ? __uint_as_float(uint32_t(__ldg(q + i)) << 16) : 0.0f;
    }
  } else {
    const float* q = reinterpret_cast<const float*>(p);
    if (vec && n == 16) {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(q) + h);
        v[4 * h] = t.x; v[4 * h + 1] = t.y; v[4 * h + 2] = t.z; v[4 * h + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = i < n ? __ldg(q + i) : 0.0f;
    }
  }
}

// Work item = (group of nb 16-pixel blocks, tap (i, j), 256-channel tile).
template <typename T, int MODE, int BM, bool FAST>
__device__ __forceinline__ void im2col_body(const ConvArgs& a, const Quant& q, float* tile,
                                            uint8_t* cbuf, int cstride, Stat& st) {
  const uint32_t bitmap = BM ? uint32_t(BM) : a.bitmap;
  const int rank = BM ? __builtin_popcount(uint32_t(BM)) : a.rank;
  const int tid = threadIdx.x;
  const int pr = tid >> 4, pb = tid & 15;
  const T* x = static_cast<const T*>(a.x);
  const int taps = a.k * a.k;
  const int total_blocks = a.B * a.nblk;
  for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
    const int ct = item % a.ctiles;
    const int rest = item / a.ctiles;
    const int tap = rest % taps;
    const int g = rest / taps;
    const int ti = tap / a.k, tj = tap - ti * a.k;
    const int c0 = ct * kCols;
    const int gb0 = g * a.nb;
    const int nbl = min(a.nb, total_blocks - gb0);
    for (int bl = 0; bl < nbl; ++bl) {
      const int gb = gb0 + bl;
      const int s = gb / a.nblk;
      const int blk = gb - s * a.nblk;
      // phase 1: gather this thread's 16 channels of output pixel l for tap (ti, tj)
      {
        const int l = blk * 16 + pr;
        const int c = c0 + pb * 16;
        int n = 0;
        const T* p = x;
        if (l < a.L && c < a.C) {
          const int ho = l / a.Wo, wo = l - ho * a.Wo;
          const int h = ho * a.stride - a.pad + ti, w = wo * a.stride - a.pad + tj;
          if (h >= 0 && h < a.H && w >= 0 && w < a.W) {
            n = min(16, a.C - c);
            p = x + ((int64_t(s) * a.H + h) * a.W + w) * a.C + c;
          }
        }
        float v[16];
        load16<T>(p, n, a.vec, v);
        float* row = tile + pr * (kCols + 4);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          *reinterpret_cast<float4*>(row + pb * 16 + 4 * q4) =
              make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
      }
      __syncthreads();
      // phase 2: channel pair (2t, 2t+1): projection along the 16 pixels
      if (tid < kCols / 2) {
        const int cc = 2 * tid;
        if (c0 + cc < a.C) {
          float2 pv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) pv[i] = *reinterpret_cast<const float2*>(tile + i * (kCols + 4) + cc);
          fwht16_pair(pv);
          if (MODE == kStats) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if ((bitmap >> i) & 1u) st.add2(pv[i].x, pv[i].y);
          } else {
            uint8_t* ox = cbuf + cc * cstride + bl * rank;
            uint8_t* oy = ox + cstride;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if ((bitmap >> i) & 1u) {
                const int j = BM ? __builtin_popcount(uint32_t(BM) & ((1u << i) - 1u))
                                 : __popc(bitmap & ((1u << i) - 1u));
                const uint32_t pq = quant2<FAST>(pv[i], q);
                ox[j] = uint8_t(pq & 0xFFu);
                oy[j] = uint8_t((pq >> 16) & 0xFFu);
              }
            }
          }
        }
      }
      __syncthreads();
    }
    if (MODE == kQuant) {
      // flush: channel c of this tap is payload row c*k*k + tap
      const int run = nbl * rank;
      const int64_t k0 = int64_t(gb0) * rank;
      const int nc = min(kCols, a.C - c0);
      for (int i = tid; i < nc * run; i += kThreads) {
        const int c = i / run, o = i - c * run;
        a.dst[(int64_t(c0 + c) * taps + tap) * a.ld_dst + k0 + o] = int8_t(cbuf[c * cstride + o]);
      }
      __syncthreads();
    }
  }
}

template <typename T, int MODE, int BM>
__global__ void __launch_bounds__(kThreads) im2col_proj_kernel(ConvArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  float* tile = reinterpret_cast<float*>(smem);  // 16 x (256 + 4) fp32
  uint8_t* cbuf = smem + 16 * (kCols + 4) * sizeof(float);
  const int cstride = a.nb * (BM ? __builtin_popcount(uint32_t(BM)) : a.rank) + 16;
  Stat st;
  if (MODE == kStats) {
    Quant dummy{};
    im2col_body<T, MODE, BM, true>(a, dummy, tile, cbuf, cstride, st);
    st.warp_reduce();
    if ((threadIdx.x & 31) == 0) st.commit(a.stats + 2);
    return;
  }
  const Quant q = make_quant(a.stats + 2, a.bits);
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.scale) *a.scale = q.s;
  if (blockIdx.x == 0 && threadIdx.x == 0) flag_nonfinite(q, a.nonfinite);
  if (q.fast)
    im2col_body<T, MODE, BM, true>(a, q, tile, cbuf, cstride, st);
  else
    im2col_body<T, MODE, BM, false>(a, q, tile, cbuf, cstride, st);
}

template <typename T, int MODE>
void launch_im2col_mode(const ConvArgs& a, cudaStream_t st) {
  const size_t smem = 16 * (kCols + 4) * sizeof(float) + size_t(kCols) * (a.nb * a.rank + 16);
  const int grid = a.items < num_sms() * 4 ? a.items : num_sms() * 4;
  switch (a.bitmap) {
    case 0x5555:
      cudaFuncSetAttribute(im2col_proj_kernel<T, MODE, 0x5555>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      im2col_proj_kernel<T, MODE, 0x5555><<<grid, kThreads, smem, st>>>(a);
      break;
    default:
      cudaFuncSetAttribute(im2col_proj_kernel<T, MODE, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      im2col_proj_kernel<T, MODE, 0><<<grid, kThreads, smem, st>>>(a);
      break;
  }
}

// ------------------------------------------------------------------ col2im
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(256) col2im_kernel(const TIn* __restrict__ dcols, int64_t ld,
                                                     int B, int H, int W, int C, int k, int stride,
                                                     int pad, int Ho, int Wo, TOut* __restrict__ dx) {
  const int64_t total = int64_t(B) * H * W * C;
  const int taps = k * k;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(e % C);
    int64_t r = e / C;
    const int w = int(r % W);
    r /= W;
    const int h = int(r % H);
    const int b = int(r / H);
    float acc = 0.0f;
    for (int i = 0; i < k; ++i) {
      const int hh = h + pad - i;
      if (hh < 0 || hh % stride) continue;
      const int ho = hh / stride;
      if (ho >= Ho) continue;
      for (int j = 0; j < k; ++j) {
        const int ww = w + pad - j;
        if (ww < 0 || ww % stride) continue;
        const int wo = ww / stride;
        if (wo >= Wo) continue;
        const int64_t row = int64_t(b) * Ho * Wo + ho * Wo + wo;
        float v;
        if (sizeof(TIn) == 2)
          v = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(dcols)[row * ld + c * taps + i * k + j]);
        else
          v = reinterpret_cast<const float*>(dcols)[row * ld + c * taps + i * k + j];
        acc = __fadd_rn(acc, v);  // (i, j) order = the reference's scatter-add order
      }
    }
    if (sizeof(TOut) == 2)
      reinterpret_cast<__nv_bfloat16*>(dx)[e] = __float2bfloat16_rn(acc);
    else
      reinterpret_cast<float*>(dx)[e] = acc;
  }
}

// Tap-major variant: dcols columns ordered (tap, c) (the W codes rows permuted
// tap-major before the dX GEMM), so each tap's C channels are contiguous: a
// thread owns 8 channels of one output pixel, 16-byte loads per tap, fp32 sums
// in the reference's (i, j) order (the per-element summation order, and so the
// result, is the same as col2im_kernel's).
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(256) col2im_tapmajor_kernel(const TIn* __restrict__ dcols, int64_t ld, int B,
                                                              int H, int W, int C, int k, int stride, int pad,
                                                              int Ho, int Wo, TOut* __restrict__ dx) {
  const int groups = C >> 3;
  const int64_t total = int64_t(B) * H * W * groups;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int c0 = int(e % groups) * 8;
    int64_t r = e / groups;
    const int w = int(r % W);
    r /= W;
    const int h = int(r % H);
    const int b = int(r / H);
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
    for (int i = 0; i < k; ++i) {
      const int hh = h + pad - i;
      if (hh < 0 || hh % stride) continue;
      const int ho = hh / stride;
      if (ho >= Ho) continue;
      for (int j = 0; j < k; ++j) {
        const int ww = w + pad - j;
        if (ww < 0 || ww % stride) continue;
        const int wo = ww / stride;
        if (wo >= Wo) continue;
        const int64_t row = int64_t(b) * Ho * Wo + ho * Wo + wo;
        const TIn* src = dcols + row * ld + int64_t(i * k + j) * C + c0;
        float v[8];
        if (sizeof(TIn) == 2) {
          const uint4 t = __ldg(reinterpret_cast<const uint4*>(src));
          const uint32_t u[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            v[2 * q] = __uint_as_float(u[q] << 16);
            v[2 * q + 1] = __uint_as_float(u[q] & 0xFFFF0000u);
          }
        } else {
          const float4 t0 = __ldg(reinterpret_cast<const float4*>(src));
          const float4 t1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
          v[0] = t0.x; v[1] = t0.y; v[2] = t0.z; v[3] = t0.w;
          v[4] = t1.x; v[5] = t1.y; v[6] = t1.z; v[7] = t1.w;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], v[q]);
      }
    }
    const int64_t o = ((int64_t(b) * H + h) * W + w) * C + c0;
    if (sizeof(TOut) == 2) {
      uint32_t u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        __nv_bfloat162 t = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
        u[q] = *reinterpret_cast<uint32_t*>(&t);
      }
      *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dx) + o) = make_uint4(u[0], u[1], u[2], u[3]);
    } else {
      float* d = reinterpret_cast<float*>(dx) + o;
      *reinterpret_cast<float4*>(d) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      *reinterpret_cast<float4*>(d + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
  }
}

}  // namespace

bool launch_col2im_tapmajor(const void* dcols, int in_dtype, int64_t ld, int B, int H, int W, int C, int k,
                            int stride, int pad, void* dx, int out_dtype, cudaStream_t st) {
  const size_t ein = in_dtype == kBF16 ? 2 : 4, eout = out_dtype == kBF16 ? 2 : 4;
  if (C % 8 || (reinterpret_cast<uintptr_t>(dcols) % 16) || (ld * ein) % 16 ||
      (reinterpret_cast<uintptr_t>(dx) % 16) || (size_t(C) * eout) % 16)
    return false;
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  const int64_t total = int64_t(B) * H * W * (C / 8);
  const int64_t want = (total + 255) / 256;
  const int grid = int(want < num_sms() * 16 ? want : num_sms() * 16);
  if (in_dtype == kBF16 && out_dtype == kBF16)
    col2im_tapmajor_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(dcols), ld, B, H, W, C, k, stride, pad, Ho, Wo,
        static_cast<__nv_bfloat16*>(dx));
  else if (in_dtype == kBF16)
    col2im_tapmajor_kernel<__nv_bfloat16, float><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(dcols), ld, B, H, W, C, k, stride, pad, Ho, Wo, static_cast<float*>(dx));
  else if (out_dtype == kBF16)
    col2im_tapmajor_kernel<float, __nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const float*>(dcols), ld, B, H, W, C, k, stride, pad, Ho, Wo, static_cast<__nv_bfloat16*>(dx));
  else
    col2im_tapmajor_kernel<float, float><<<grid, 256, 0, st>>>(static_cast<const float*>(dcols), ld, B, H, W, C, k,
                                                                stride, pad, Ho, Wo, static_cast<float*>(dx));
  return true;
}

void launch_im2col_proj(const void* x, int dtype, int B, int H, int W, int C, int k, int stride,
                        int pad, uint32_t bitmap, int bits, int mode, uint32_t* stats, int8_t* dst,
                        int64_t ld_dst, float* scale, cudaStream_t st) {
  ConvArgs a{};
  a.nonfinite = nonfinite_word();
  a.x = x;
  a.B = B; a.H = H; a.W = W; a.C = C; a.k = k; a.stride = stride; a.pad = pad;
  a.Ho = (H + 2 * pad - k) / stride + 1;
  a.Wo = (W + 2 * pad - k) / stride + 1;
  a.L = a.Ho * a.Wo;
  a.nblk = (a.L + 15) / 16;
  a.rank = __builtin_popcount(bitmap);
  a.bits = bits;
  a.bitmap = bitmap;
  a.ctiles = (C + kCols - 1) / kCols;
  const int total_blocks = B * a.nblk;
  a.nb = a.rank >= 8 ? 4 : (a.rank >= 4 ? 8 : 16);
  while (a.nb > 1 && ((total_blocks + a.nb - 1) / a.nb) * k * k * a.ctiles < num_sms() * 4) a.nb >>= 1;
  a.items = ((total_blocks + a.nb - 1) / a.nb) * k * k * a.ctiles;
  a.stats = stats;
  a.dst = dst;
  a.ld_dst = ld_dst;
  a.scale = scale;
  const size_t esz = dtype == kBF16 ? 2 : 4;
  a.vec = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && ((size_t(C) * esz) % 16 == 0);
  if (dtype == kBF16) {
    if (mode == kStats) launch_im2col_mode<__nv_bfloat16, kStats>(a, st);
    else launch_im2col_mode<__nv_bfloat16, kQuant>(a, st);
  } else {
    if (mode == kStats) launch_im2col_mode<float, kStats>(a, st);
    else launch_im2col_mode<float, kQuant>(a, st);
  }
}

void launch_col2im(const void* dcols, int in_dtype, int64_t ld, int B, int H, int W, int C, int k,
                   int stride, int pad, void* dx, int out_dtype, cudaStream_t st) {
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  const int64_t total = int64_t(B) * H * W * C;
  const int64_t want = (total + 255) / 256;
  const int grid = int(want < num_sms() * 16 ? want : num_sms() * 16);
  if (in_dtype == kBF16 && out_dtype == kBF16)
    col2im_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(dcols), ld, B, H, W, C, k, stride, pad, Ho, Wo,
        static_cast<__nv_bfloat16*>(dx));
  else if (in_dtype == kBF16)
    col2im_kernel<__nv_bfloat16, float><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(dcols), ld, B, H, W, C, k, stride, pad, Ho, Wo,
        static_cast<float*>(dx));
  else if (out_dtype == kBF16)
    col2im_kernel<float, __nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const float*>(dcols), ld, B, H, W, C, k, stride, pad, Ho, Wo,
        static_cast<__nv_bfloat16*>(dx));
  else
    col2im_kernel<float, float><<<grid, 256, 0, st>>>(static_cast<const float*>(dcols), ld, B, H, W,
                                                      C, k, stride, pad, Ho, Wo,
                                                      static_cast<float*>(dx));
}

}  // namespace hlq
