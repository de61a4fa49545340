// Block-Hadamard transform + per-tensor amax + pseudo-stochastic quantizer.
//
// Operands of the HLQ backward, all produced here:
//   gx left   Q4(HT_O(gy))   HT along the contiguous axis, codes (T, pad16(O))  backprop.py:362,367
//   gx right  Q4(HT_O(W))    HT along rows of W, codes written (I, pad16(O))    backprop.py:363,368
//   gw left   Q8(P gy)^T     rank-r projection along tokens, codes (O, K)       backprop.py:401-407
//   gw right  Q8(P X)        ACBP, rank-r projection along tokens, (I, K)       backprop.py:373-385
// Everything the tensor-core GEMM consumes is written K-major.
//
// One kernel template (tile_kernel) covers all of them.  A CTA owns NB
// consecutive 16-row projection blocks x 256 columns of a (S segments x R rows
// x C cols) view.  Per block:
//   phase 1: thread (row r, 16-col block b) loads 16 contiguous elements
//            (128-bit loads), runs the column-direction FWHT in registers (gx
//            operand) and parks the raw values in shared memory (swizzled);
//   phase 2: thread c reads its column's 16 rows from shared memory, runs the
//            row-direction FWHT and keeps the plan's bases (gw operand / W);
//            codes are staged in shared memory and written as >=32-byte runs.
// gy is therefore read once per pass for BOTH products (the "dual" mode).
//
// Two passes: STATS (max|w| and min nonzero |w| of the transformed values,
// one atomicMax per CTA per statistic, on the IEEE bits) then QUANT.
//
// Bit-exactness (hadamard.py:121-134, quantize.py:94-145):
//  * butterfly stages h = 1, 2, 4, 8, (lower, upper) = (a + b, a - b), fp32 RN;
//  * the reference multiplies by 0.25 then divides by s; we keep w = 4v and
//    divide by d = s/512, i.e. compute Q = RN(w/d) = 2048 * RN(v/s) exactly
//    (power-of-two rescalings are exact for normal numbers), with the
//    reciprocal-FMA division Q = fma(fma(-Q0, d, w), r, Q0), r = RN(1/d),
//    Q0 = RN(w r) -- verified equal to IEEE division on 2.8e9 pairs inside the
//    guard |w| >= 2^-100, |Q| >= 2^-100, 2^-125 < d < 2^125
//    (tools/verify_fast_div.c).  The STATS pass records min nonzero |w| so the
//    QUANT pass can check the guard once per tensor and otherwise fall back to
//    the literal IEEE-division formula;
//  * floor(q), frac(q) and the up-decision use no conversion instructions:
//    F = floor(Q), C = ceil(Q) come from the bit patterns of Q + 1.5*2^23
//    rounded down / up, lo = F >> 11, frac*2048 > u  <=>  C - 2048*lo > u;
//  * the draw u = bits(v) & 0x7FF equals bits(w) & 0x7FF (same mantissa).
#include <cuda_bf16.h>
#include <cstdint>

#include "hlq_internal.h"
#include "hlq_ptx.cuh"

namespace hlq {

namespace {

constexpr int kTileCols = 256;
constexpr int kThreads = 256;
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr int kMagicShift = 0x4B400000 >> 11;

// ------------------------------------------------------------------ loads
// 16 consecutive elements -> fp32.  `n` valid (0..16); vector path if aligned.
__device__ __forceinline__ void load16(const float* p, int n, bool vec, float (&v)[16]) {
  if (vec && n == 16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p) + q);
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = i < n ? __ldg(p + i) : 0.0f;
  }
}
__device__ __forceinline__ void load16(const __nv_bfloat16* p, int n, bool vec, float (&v)[16]) {
  if (vec && n == 16) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint4 t = __ldg(reinterpret_cast<const uint4*>(p) + q);
      const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[8 * q + 2 * k] = __uint_as_float(w[k] << 16);
        v[8 * q + 2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
      }
    }
  } else {
    const unsigned short* q = reinterpret_cast<const unsigned short*>(p);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = i < n ? __uint_as_float(uint32_t(__ldg(q + i)) << 16) : 0.0f;
  }
}

// ------------------------------------------------------------------ transform
// Un-normalised 16-point FWHT (the 0.25 is folded into the quantizer divisor).
__device__ __forceinline__ void fwht16_raw(float (&v)[16]) {
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
}

// ------------------------------------------------------------------ statistics
struct Stat {
  uint32_t amax = 0;             // max |w| bits (NaN/Inf land >= 0x7F800000)
  uint32_t minnz = 0xFFFFFFFFu;  // min (|w| bits - 1): the smallest nonzero magnitude
  __device__ __forceinline__ void add(float w) {
    const uint32_t a = __float_as_uint(w) & 0x7FFFFFFFu;
    amax = max(amax, a);
    minnz = min(minnz, a - 1u);
  }
};

// stats layout in global memory: {amax, ~minnz} per operand, both reduced with
// atomicMax so a zero memset is the identity.
__device__ __forceinline__ void reduce_stat_to_global(Stat s, uint32_t* g) {
  __shared__ uint32_t red[2][kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s.amax = max(s.amax, __shfl_xor_sync(0xffffffffu, s.amax, o));
    s.minnz = min(s.minnz, __shfl_xor_sync(0xffffffffu, s.minnz, o));
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) { red[0][w] = s.amax; red[1][w] = s.minnz; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a = 0, m = 0xFFFFFFFFu;
    for (int i = 0; i < kThreads / 32; ++i) { a = max(a, red[0][i]); m = min(m, red[1][i]); }
    if (a) atomicMax(g, a);
    if (~m) atomicMax(g + 1, ~m);
  }
}

// ------------------------------------------------------------------ quantizer
struct Quant {
  float s, d, r, lim, qmax;
  bool fast;
};

// scale = f32(amax_v) / f32(qmax), 0 -> 1 (quantize.py:94-100), amax_v = RN(0.25 * max|w|),
// which equals max|RN(0.25 w)| because rounding is monotone.
__device__ __forceinline__ Quant make_quant(const uint32_t* g, int bits) {
  Quant q;
  q.qmax = float((1 << (bits - 1)) - 1);
  const float amax_w = __uint_as_float(g[0]);
  const float amax_v = __fmul_rn(amax_w, 0.25f);
  float s = __fdiv_rn(amax_v, q.qmax);
  if (s == 0.0f) s = 1.0f;
  q.s = s;
  q.d = __fmul_rn(s, 1.0f / 512.0f);
  q.r = __frcp_rn(q.d);
  q.lim = 2048.0f * q.qmax;
  const uint32_t inv = g[1];
  const float minnz = inv ? __uint_as_float(~inv + 1u) : 0.0f;  // 0: no nonzero value at all
  q.fast = (g[0] < 0x7F800000u) && s > 0x1p-116f &&
           (minnz == 0.0f || (minnz >= 0x1p-100f && minnz >= __fmul_rn(s, 0x1p-108f)));
  return q;
}

__device__ __forceinline__ int quant_fast(float w, const Quant& q) {
  float Q = __fmul_rn(w, q.r);
  const float e = __fmaf_rn(-Q, q.d, w);
  Q = __fmaf_rn(e, q.r, Q);
  Q = fminf(fmaxf(Q, -q.lim), q.lim);
  const int Fb = __float_as_int(__fadd_rd(Q, kMagic));
  const int Cb = __float_as_int(__fadd_ru(Q, kMagic));
  const int u = __float_as_int(w) & 0x7FF;
  const int up = (Cb - (Fb & ~2047)) > u ? 1 : 0;
  return (Fb >> 11) - kMagicShift + up;
}

// Literal restatement of quantize.py:140-145 (IEEE division), used when the
// fast path's guard fails for the tensor.
__device__ __forceinline__ int quant_exact(float w, const Quant& q) {
  const float v = __fmul_rn(w, 0.25f);
  const float qq = __fdiv_rn(v, q.s);
  const float lo = floorf(qq);
  const float draw = __uint2float_rn(__float_as_uint(v) & 0x7FFu);
  const float frac = __fmul_rn(__fsub_rn(qq, lo), 2048.0f);
  float c = __fadd_rn(lo, frac > draw ? 1.0f : 0.0f);
  c = fminf(fmaxf(c, -q.qmax), q.qmax);
  return static_cast<int>(c);
}

template <bool FAST>
__device__ __forceinline__ int quant(float w, const Quant& q) {
  return FAST ? quant_fast(w, q) : quant_exact(w, q);
}

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return (uint32_t(a) & 0xFFu) | ((uint32_t(b) & 0xFFu) << 8) | ((uint32_t(c) & 0xFFu) << 16) |
         (uint32_t(d) << 24);
}

// ------------------------------------------------------------------ the tile kernel
struct TileArgs {
  const void* src;
  int64_t segs, rows, cols, ld_src, seg_src;
  int64_t nblk;          // ceil(rows / 16)
  int64_t total_blocks;  // segs * nblk
  int nb;                // projection blocks per CTA
  uint32_t bitmap;
  int rank;
  int bits_gx, bits_gw;
  uint32_t* stats;  // [0,1] gx, [2,3] gw
  int8_t* dst_gx;
  int64_t ld_gx;
  int8_t* dst_gw;
  int64_t ld_gw;
  float* scale_gx;
  float* scale_gw;
  bool vec;
};

__device__ __forceinline__ int phys_col(int c) {
  // 16-float blocks split into 4 chunks, chunk index xor-swizzled by (block >> 1) & 3
  return (c & ~15) | ((((c >> 2) & 3) ^ ((c >> 5) & 3)) << 2) | (c & 3);
}

template <typename T, int MODE, bool GX, bool GW, bool FAST_GX, bool FAST_GW>
__device__ __forceinline__ void tile_body(const TileArgs& a, const Quant& qx, const Quant& qw,
                                          float* tile, uint8_t* cbuf, int cstride, Stat& sx,
                                          Stat& sw) {
  const T* src = static_cast<const T*>(a.src);
  const int64_t ncol_tiles = (a.cols + kTileCols - 1) / kTileCols;
  const int64_t ngroups = (a.total_blocks + a.nb - 1) / a.nb;
  const int64_t items = ngroups * ncol_tiles;
  const int tid = threadIdx.x;
  const int pr = tid >> 4, pb = tid & 15;  // phase-1 role: row within block, 16-col block
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t g = item / ncol_tiles;
    const int64_t ct = item - g * ncol_tiles;
    const int64_t col0 = ct * kTileCols;
    const int64_t gb0 = g * a.nb;
    const int nbl = int(a.total_blocks - gb0 < a.nb ? a.total_blocks - gb0 : a.nb);
    for (int bl = 0; bl < nbl; ++bl) {
      const int64_t gb = gb0 + bl;
      const int64_t s = gb / a.nblk;
      const int64_t blk = gb - s * a.nblk;
      // ---------------- phase 1: row pieces
      {
        const int64_t row = blk * 16 + pr;
        const int64_t c = col0 + pb * 16;
        const bool row_ok = row < a.rows;
        const int64_t cvalid = a.cols - c;
        const int n = row_ok ? int(cvalid < 0 ? 0 : (cvalid > 16 ? 16 : cvalid)) : 0;
        float v[16];
        load16(src + (n ? s * a.seg_src + row * a.ld_src + c : 0), n, a.vec, v);
        if (GW) {
          float* dstp = tile + pr * kTileCols;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int pc = phys_col(pb * 16 + 4 * q);
            *reinterpret_cast<float4*>(dstp + pc) =
                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
        if (GX && row_ok && cvalid > 0) {
          fwht16_raw(v);
          if (MODE == kStats) {
#pragma unroll
            for (int i = 0; i < 16; ++i) sx.add(v[i]);
          } else {
            uint4 p;
            p.x = pack4(quant<FAST_GX>(v[0], qx), quant<FAST_GX>(v[1], qx),
                        quant<FAST_GX>(v[2], qx), quant<FAST_GX>(v[3], qx));
            p.y = pack4(quant<FAST_GX>(v[4], qx), quant<FAST_GX>(v[5], qx),
                        quant<FAST_GX>(v[6], qx), quant<FAST_GX>(v[7], qx));
            p.z = pack4(quant<FAST_GX>(v[8], qx), quant<FAST_GX>(v[9], qx),
                        quant<FAST_GX>(v[10], qx), quant<FAST_GX>(v[11], qx));
            p.w = pack4(quant<FAST_GX>(v[12], qx), quant<FAST_GX>(v[13], qx),
                        quant<FAST_GX>(v[14], qx), quant<FAST_GX>(v[15], qx));
            *reinterpret_cast<uint4*>(a.dst_gx + (s * a.rows + row) * a.ld_gx + c) = p;
          }
        }
      }
      if (!GW) continue;
      __syncthreads();
      // ---------------- phase 2: column pieces (projection along rows)
      {
        const int64_t c = col0 + tid;
        if (c < a.cols) {
          float v[16];
          const int pc = phys_col(tid);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = tile[i * kTileCols + pc];
          fwht16_raw(v);
          if (MODE == kStats) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if ((a.bitmap >> i) & 1u) sw.add(v[i]);
          } else {
            uint8_t* out = cbuf + tid * cstride + bl * a.rank;
            uint32_t w4[4] = {0, 0, 0, 0};
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if ((a.bitmap >> i) & 1u) {
                const int j = __popc(a.bitmap & ((1u << i) - 1u));
                const uint32_t code = uint32_t(quant<FAST_GW>(v[i], qw)) & 0xFFu;
                // j is uniform across the grid; the switch keeps w4 in registers
                switch (j >> 2) {
                  case 0: w4[0] |= code << (8 * (j & 3)); break;
                  case 1: w4[1] |= code << (8 * (j & 3)); break;
                  case 2: w4[2] |= code << (8 * (j & 3)); break;
                  default: w4[3] |= code << (8 * (j & 3)); break;
                }
              }
            }
            if (a.rank == 16) {
              *reinterpret_cast<uint4*>(out) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            } else if (a.rank == 8) {
              *reinterpret_cast<uint2*>(out) = make_uint2(w4[0], w4[1]);
            } else if (a.rank == 4) {
              *reinterpret_cast<uint32_t*>(out) = w4[0];
            } else {
              for (int j = 0; j < a.rank; ++j) out[j] = uint8_t(w4[j >> 2] >> (8 * (j & 3)));
            }
          }
        }
      }
      __syncthreads();
    }
    // ---------------- write the staged projection codes: (cols, K) K-major
    if (GW && MODE == kQuant) {
      const int run = nbl * a.rank;  // contiguous bytes per column
      const int64_t k0 = gb0 * a.rank;
      const int ncols = int(a.cols - col0 < kTileCols ? a.cols - col0 : kTileCols);
      if ((run & 15) == 0 && (k0 & 15) == 0) {
        const int chunks = run >> 4;
        for (int i = tid; i < ncols * chunks; i += kThreads) {
          const int c = i / chunks, p = i - c * chunks;
          *reinterpret_cast<uint4*>(a.dst_gw + (col0 + c) * a.ld_gw + k0 + 16 * p) =
              *reinterpret_cast<const uint4*>(cbuf + c * cstride + 16 * p);
        }
      } else if ((run & 7) == 0 && (k0 & 7) == 0) {
        const int chunks = run >> 3;
        for (int i = tid; i < ncols * chunks; i += kThreads) {
          const int c = i / chunks, p = i - c * chunks;
          *reinterpret_cast<uint2*>(a.dst_gw + (col0 + c) * a.ld_gw + k0 + 8 * p) =
              *reinterpret_cast<const uint2*>(cbuf + c * cstride + 8 * p);
        }
      } else {
        for (int i = tid; i < ncols * run; i += kThreads) {
          const int c = i / run, p = i - c * run;
          a.dst_gw[(col0 + c) * a.ld_gw + k0 + p] = int8_t(cbuf[c * cstride + p]);
        }
      }
      __syncthreads();
    }
  }
}

template <typename T, int MODE, bool GX, bool GW>
__global__ void __launch_bounds__(kThreads) tile_kernel(TileArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  float* tile = reinterpret_cast<float*>(smem);  // 16 x 256 fp32
  uint8_t* cbuf = smem + (GW ? 16 * kTileCols * sizeof(float) : 0);
  const int cstride = a.nb * a.rank + 16;
  Stat sx, sw;
  if (MODE == kStats) {
    Quant dummy{};
    tile_body<T, MODE, GX, GW, true, true>(a, dummy, dummy, tile, cbuf, cstride, sx, sw);
    if (GX) reduce_stat_to_global(sx, a.stats);
    if (GW) reduce_stat_to_global(sw, a.stats + 2);
    return;
  }
  Quant qx{}, qw{};
  if (GX) qx = make_quant(a.stats, a.bits_gx);
  if (GW) qw = make_quant(a.stats + 2, a.bits_gw);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (GX && a.scale_gx) *a.scale_gx = qx.s;
    if (GW && a.scale_gw) *a.scale_gw = qw.s;
  }
  const bool fx = !GX || qx.fast, fw = !GW || qw.fast;  // uniform across the grid
  if (fx && fw)
    tile_body<T, MODE, GX, GW, true, true>(a, qx, qw, tile, cbuf, cstride, sx, sw);
  else if (fx)
    tile_body<T, MODE, GX, GW, true, false>(a, qx, qw, tile, cbuf, cstride, sx, sw);
  else if (fw)
    tile_body<T, MODE, GX, GW, false, true>(a, qx, qw, tile, cbuf, cstride, sx, sw);
  else
    tile_body<T, MODE, GX, GW, false, false>(a, qx, qw, tile, cbuf, cstride, sx, sw);
}

template <typename T, int MODE, bool GX, bool GW>
void launch_tile(const TileArgs& a, cudaStream_t stream) {
  const int64_t ncol_tiles = (a.cols + kTileCols - 1) / kTileCols;
  const int64_t ngroups = (a.total_blocks + a.nb - 1) / a.nb;
  const int64_t items = ngroups * ncol_tiles;
  const size_t smem =
      GW ? 16 * kTileCols * sizeof(float) + size_t(kTileCols) * (a.nb * a.rank + 16) : 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tile_kernel<T, MODE, GX, GW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         64 * 1024);
    attr = true;
  }
  const int64_t cap = int64_t(num_sms()) * 6;
  const int grid = int(items < 1 ? 1 : (items > cap ? cap : items));
  tile_kernel<T, MODE, GX, GW><<<grid, kThreads, smem, stream>>>(a);
}

template <typename T>
void launch_tile_modes(const TileArgs& a, int mode, bool gx, bool gw, cudaStream_t st) {
  if (mode == kStats) {
    if (gx && gw) launch_tile<T, kStats, true, true>(a, st);
    else if (gx) launch_tile<T, kStats, true, false>(a, st);
    else launch_tile<T, kStats, false, true>(a, st);
  } else {
    if (gx && gw) launch_tile<T, kQuant, true, true>(a, st);
    else if (gx) launch_tile<T, kQuant, true, false>(a, st);
    else launch_tile<T, kQuant, false, true>(a, st);
  }
}

// Blocks per CTA: >= 32-byte output runs per column when the problem is large,
// while keeping >= ~4 CTAs per SM of work.
int choose_nb(int64_t total_blocks, int64_t cols, int rank) {
  int nb = rank >= 8 ? 4 : (rank >= 4 ? 8 : 16);
  const int64_t ncol_tiles = (cols + kTileCols - 1) / kTileCols;
  while (nb > 1 && ((total_blocks + nb - 1) / nb) * ncol_tiles < int64_t(num_sms()) * 4) nb >>= 1;
  return nb;
}

}  // namespace

void launch_transform(const TransformArgs& t, int mode, cudaStream_t stream) {
  TileArgs a{};
  a.src = t.src;
  a.segs = t.segs;
  a.rows = t.rows;
  a.cols = t.cols;
  a.ld_src = t.ld_src;
  a.seg_src = t.seg_src;
  a.nblk = (t.rows + 15) / 16;
  a.total_blocks = t.segs * a.nblk;
  a.bitmap = t.bitmap;
  a.rank = t.do_gw ? __builtin_popcount(t.bitmap) : 0;
  a.bits_gx = t.bits_gx;
  a.bits_gw = t.bits_gw;
  a.stats = t.stats;
  a.dst_gx = t.dst_gx;
  a.ld_gx = t.ld_gx;
  a.dst_gw = t.dst_gw;
  a.ld_gw = t.ld_gw;
  a.scale_gx = t.scale_gx;
  a.scale_gw = t.scale_gw;
  const size_t esz = t.dtype == kBF16 ? 2 : 4;
  a.vec = (reinterpret_cast<uintptr_t>(t.src) % 16 == 0) && ((t.ld_src * esz) % 16 == 0) &&
          ((t.seg_src * esz) % 16 == 0);
  a.nb = t.do_gw ? choose_nb(a.total_blocks, t.cols, a.rank) : 4;
  if (t.dtype == kBF16)
    launch_tile_modes<__nv_bfloat16>(a, mode, t.do_gx, t.do_gw, stream);
  else
    launch_tile_modes<float>(a, mode, t.do_gx, t.do_gw, stream);
}

}  // namespace hlq
