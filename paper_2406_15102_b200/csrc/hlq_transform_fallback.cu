// Register-pipelined fallback of the transform kernels (hlq_transform.cu), used
// when the source cannot be described by a TMA tensor map (unaligned base or
// row stride).  Same numerics, same outputs.
//
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
// x C cols) view, one block ("step") at a time:
//   phase 1: thread (row r, 16-col block b) holds 16 contiguous elements in
//            registers (128-bit loads, issued two steps ahead), runs the
//            column-direction FWHT (gx operand) and parks the raw bytes in a
//            double-buffered, bank-swizzled shared tile;
//   phase 2: thread c reads the 16 rows of columns (2c, 2c+1) from shared
//            memory and runs the row-direction FWHT with packed f32x2 math,
//            keeping only the plan's bases (dead butterflies are pruned for the
//            common compile-time basis sets); codes are staged in shared
//            memory and written as >= 32-byte runs per output row.
// gy is therefore read once per pass for BOTH products (the "dual" mode).
//
// Two passes: STATS (max|w| and min nonzero |w| of the transformed values,
// one atomicMax per CTA per statistic, on the IEEE bits) then QUANT.
//
// Bit-exactness (hadamard.py:121-134, quantize.py:94-145):
//  * butterfly stages h = 1, 2, 4, 8, (lower, upper) = (a + b, a - b), fp32 RN
//    (pairing two independent lanes in one f32x2 op changes nothing per lane);
//  * the reference multiplies by 0.25 then divides by s.  We keep w = 4v and
//    divide by d = s/512, i.e. compute Q = RN(w/d) = 2048 * RN(v/s) exactly
//    (power-of-two rescalings are exact for normal numbers) with the
//    reciprocal-FMA division Q = fma(fma(-Q0, d, w), r, Q0), r = RN(1/d),
//    Q0 = RN(w r) -- verified equal to IEEE division on 2.8e9 pairs inside the
//    guard |w| >= 2^-100, |Q| >= 2^-100, 2^-125 < d < 2^125
//    (tools/verify_fast_div.c).  The STATS pass records min nonzero |w| so the
//    QUANT pass checks the guard once per tensor and otherwise falls back to
//    the literal IEEE-division formula;
//  * code = lo + [frac*2048 > u] = ceil((Q - u) / 2048) exactly, evaluated as
//    RU(RU(Q - u) * 2^-11 + 1.5*2^23): the low byte of that float's bit
//    pattern IS the int8 code -- no conversion instructions anywhere.  Q is
//    clamped to +-2048*qmax first, which yields the same codes as the
//    reference's clip after rounding;
//  * the draw u = bits(v) & 0x7FF equals bits(w) & 0x7FF (same mantissa).
#include <cuda_bf16.h>
#include <cstdint>

#include "hlq_internal.h"
#include "hlq_ptx.cuh"

namespace hlq {

namespace {

constexpr int kTileCols = 256;
constexpr int kThreads = 256;
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: ulp 1, integers in its low mantissa bits

// ------------------------------------------------------------------ packed fp32x2
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 f2add_rp(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rp.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// The reference's frac = RN(q - floor(q)) is RN(q + 1) for q in (-0.5, 0):
// Qr = RU(Q - 2^-14) there, Q elsewhere (one int max; see hlq_quant.cuh).
__device__ __forceinline__ float2 ref_frac_adjust(float2 Q) {
  const float2 t = f2add_rp(Q, make_float2(-0x1p-14f, -0x1p-14f));
  return make_float2(__int_as_float(max(__float_as_int(Q.x), __float_as_int(t.x))),
                     __int_as_float(max(__float_as_int(Q.y), __float_as_int(t.y))));
}
__device__ __forceinline__ float2 f2fma_rp(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rp.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// ------------------------------------------------------------------ element types
template <typename T>
struct Traits;
template <>
struct Traits<float> {
  static constexpr int kVec = 4;        // uint4 chunks per 16 elements
  static constexpr int kRowBytes = 1024;  // one 256-col smem row
};
template <>
struct Traits<__nv_bfloat16> {
  static constexpr int kVec = 2;
  static constexpr int kRowBytes = 512;
};

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// raw chunks -> 16 fp32 values
template <typename T>
__device__ __forceinline__ void unpack16(const uint4 (&raw)[Traits<T>::kVec], float (&v)[16]);
template <>
__device__ __forceinline__ void unpack16<float>(const uint4 (&raw)[4], float (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[4 * q] = __uint_as_float(raw[q].x); v[4 * q + 1] = __uint_as_float(raw[q].y);
    v[4 * q + 2] = __uint_as_float(raw[q].z); v[4 * q + 3] = __uint_as_float(raw[q].w);
  }
}
template <>
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4 (&raw)[2], float (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const uint32_t w[4] = {raw[q].x, raw[q].y, raw[q].z, raw[q].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) { v[8 * q + 2 * k] = bf_lo(w[k]); v[8 * q + 2 * k + 1] = bf_hi(w[k]); }
  }
}

// Load the 16 elements at p (n valid, zero-filled beyond) as raw 16-byte chunks.
template <typename T>
__device__ __forceinline__ void load_raw(const T* p, int n, bool vec, uint4 (&raw)[Traits<T>::kVec]) {
  constexpr int V = Traits<T>::kVec;
  if (vec && n == 16) {
#pragma unroll
    for (int q = 0; q < V; ++q) raw[q] = __ldg(reinterpret_cast<const uint4*>(p) + q);
    return;
  }
  uint32_t w[4 * V];
  if (sizeof(T) == 4) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = i < n ? __ldg(s + i) : 0u;
  } else {
    const unsigned short* s = reinterpret_cast<const unsigned short*>(p);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t lo = 2 * i < n ? uint32_t(__ldg(s + 2 * i)) : 0u;
      const uint32_t hi = 2 * i + 1 < n ? uint32_t(__ldg(s + 2 * i + 1)) : 0u;
      w[i] = lo | (hi << 16);
    }
  }
#pragma unroll
  for (int q = 0; q < V; ++q) raw[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

// ------------------------------------------------------------------ transforms
// Un-normalised 16-point FWHT of one vector (the 0.25 is folded into the
// quantizer divisor).  Register pairs (v[i], v[i+8]) run stages h = 1, 2, 4
// as f32x2; stage 8 pairs the two lanes of each register pair.
__device__ __forceinline__ void fwht16_raw(float (&v)[16]) {
  float2 p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = make_float2(v[i], v[i + 8]);
#pragma unroll
  for (int h = 1; h < 8; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (!(i & h)) {
        const float2 a = p[i], b = p[i + h];
        p[i] = f2add(a, b);
        p[i + h] = f2sub(a, b);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = __fadd_rn(p[i].x, p[i].y);
    v[i + 8] = __fsub_rn(p[i].x, p[i].y);
  }
}

// Two independent columns at once: FWHT of a[.] (lane x) and b[.] (lane y).
// Only outputs selected by KEEP (compile-time bitmap, 0 = all) are guaranteed;
// the compiler removes butterflies that feed nothing.
__device__ __forceinline__ void fwht16_pair(float2 (&p)[16]) {
#pragma unroll
  for (int h = 1; h < 16; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!(i & h)) {
        const float2 a = p[i], b = p[i + h];
        p[i] = f2add(a, b);
        p[i + h] = f2sub(a, b);
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
  bool nonfinite;
};

// scale = f32(amax_v) / f32(qmax), 0 -> 1 (quantize.py:94-100), amax_v = RN(0.25 * max|w|),
// which equals max|RN(0.25 w)| because rounding is monotone.
__device__ __forceinline__ Quant make_quant(const uint32_t* g, int bits) {
  Quant q;
  q.qmax = float((1 << (bits - 1)) - 1);
  q.nonfinite = g[0] >= 0x7F800000u;
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

// Two codes (low byte of each returned word).
__device__ __forceinline__ uint2 quant_fast2(float2 w, const Quant& q) {
  float2 Q = f2mul(w, f2(q.r));
  const float2 e = f2fma(Q, f2(-q.d), w);
  Q = ref_frac_adjust(f2fma(e, f2(q.r), Q));  // hlq_quant.cuh: the reference's RN(q - floor(q))
  Q.x = fminf(fmaxf(Q.x, -q.lim), q.lim);
  Q.y = fminf(fmaxf(Q.y, -q.lim), q.lim);
  // -u as an exact float: (2^23) - (2^23 + u)
  const float2 ub = make_float2(__uint_as_float((__float_as_uint(w.x) & 0x7FFu) | 0x4B000000u),
                                __uint_as_float((__float_as_uint(w.y) & 0x7FFu) | 0x4B000000u));
  const float2 nu = f2sub(f2(8388608.0f), ub);
  const float2 z = f2add_rp(Q, nu);
  const float2 c = f2fma_rp(z, f2(1.0f / 2048.0f), f2(kMagic));
  return make_uint2(__float_as_uint(c.x), __float_as_uint(c.y));
}

// Literal restatement of quantize.py:140-145 (IEEE division), used when the
// fast path's guard fails for the tensor.
__device__ __forceinline__ uint32_t quant_exact(float w, const Quant& q) {
  const float v = __fmul_rn(w, 0.25f);
  const float qq = __fdiv_rn(v, q.s);
  const float lo = floorf(qq);
  const float draw = __uint2float_rn(__float_as_uint(v) & 0x7FFu);
  const float frac = __fmul_rn(__fsub_rn(qq, lo), 2048.0f);
  float c = __fadd_rn(lo, frac > draw ? 1.0f : 0.0f);
  c = fminf(fmaxf(c, -q.qmax), q.qmax);
  return uint32_t(static_cast<int>(c));
}

template <bool FAST>
__device__ __forceinline__ uint2 quant2(float2 w, const Quant& q) {
  if (FAST) return quant_fast2(w, q);
  return make_uint2(quant_exact(w.x, q), quant_exact(w.y, q));
}

// low bytes of a, b, c, d -> one word
__device__ __forceinline__ uint32_t pack_bytes(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  const uint32_t ab = __byte_perm(a, b, 0x0040);   // [a0, b0, a0, a0] -> use bytes 0,1
  const uint32_t cd = __byte_perm(c, d, 0x0040);
  return __byte_perm(ab, cd, 0x5410);
}

// ------------------------------------------------------------------ the tile kernel
struct TileArgs {
  const void* src;
  int64_t segs, rows, cols, ld_src, seg_src;
  int64_t nblk;          // ceil(rows / 16)
  int64_t total_blocks;  // segs * nblk
  int nb;                // projection blocks per CTA work item
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
  uint32_t* nonfinite;  // nonfinite_word()
  bool pack_gx;         // gx codes packed int4 (two per byte, low nibble first)
  bool vec;
};

// byte offset of 16-byte chunk q of 16-col block b inside one smem row
// (xor swizzle so the 8 threads of a store phase hit 8 distinct bank groups)
template <typename T>
__device__ __forceinline__ int chunk_off(int b, int q) {
  if (Traits<T>::kVec == 2) return b * 32 + ((q ^ ((b >> 2) & 1)) << 4);
  return b * 64 + ((q ^ ((b >> 1) & 3)) << 4);
}

// One step = one 16-row block of the tile.  Precomputed per step:
struct StepPos {
  const void* ptr;  // this thread's 16 phase-1 elements
  int n;            // valid elements for this thread
  int64_t row;      // global row index (seg*rows + row) for gx output, -1 if invalid
  int col0;         // tile's first column
  int bl;           // block index inside the work item
  bool last;        // last block of the work item (flush codes after it)
  int nbl;          // blocks in this work item
  int gb0;          // first global block of the work item
  bool valid;
};

// Walks this CTA's (work item, block) steps with 32-bit counters; the only
// divisions happen once per work item.
struct StepIter {
  int item, items, ncol_tiles, nb, total_blocks, nblk;
  int bl, nbl, gb0, col0, s, blk;
  __device__ __forceinline__ void start_item() {
    if (item >= items) return;
    const int g = item / ncol_tiles;
    col0 = (item - g * ncol_tiles) * kTileCols;
    gb0 = g * nb;
    nbl = min(nb, total_blocks - gb0);
    bl = 0;
    s = gb0 / nblk;
    blk = gb0 - s * nblk;
  }
  __device__ __forceinline__ void advance() {
    if (item >= items) return;
    if (++bl == nbl) {
      item += gridDim.x;
      start_item();
    } else if (++blk == nblk) {
      blk = 0;
      ++s;
    }
  }
};

template <int BM, int MODE, bool GX, bool GW, bool FAST_GX, bool FAST_GW, typename T>
__device__ __forceinline__ void run_tile(const TileArgs& a, const Quant& qx, const Quant& qw,
                                         uint8_t* smem, Stat& sx, Stat& sw) {
  constexpr int V = Traits<T>::kVec;
  constexpr int kRow = Traits<T>::kRowBytes;
  uint8_t* tiles = smem;                           // [2][16][kRow]
  uint8_t* cbuf = smem + (GW ? 2 * 16 * kRow : 0);  // [256][cstride]
  const uint32_t bitmap = BM ? uint32_t(BM) : a.bitmap;
  const int rank = BM ? __builtin_popcount(uint32_t(BM)) : a.rank;
  const int cstride = a.nb * rank + 16;
  const int tid = threadIdx.x;
  const int pr = tid >> 4, pb = tid & 15;
  const T* src = static_cast<const T*>(a.src);
  const int rows = int(a.rows), cols = int(a.cols);

  // iterator over (item, block) steps of this CTA
  StepIter it;
  it.ncol_tiles = (cols + kTileCols - 1) / kTileCols;
  it.nb = a.nb;
  it.total_blocks = int(a.total_blocks);
  it.nblk = int(a.nblk);
  it.items = ((it.total_blocks + a.nb - 1) / a.nb) * it.ncol_tiles;
  it.item = blockIdx.x;
  it.start_item();
  auto pos_of = [&]() {
    StepPos p;
    p.valid = it.item < it.items;
    if (!p.valid) { p.ptr = src; p.n = 0; p.row = -1; p.col0 = 0; p.bl = 0; p.last = false; p.nbl = 0; p.gb0 = 0; return p; }
    p.col0 = it.col0;
    p.gb0 = it.gb0;
    p.nbl = it.nbl;
    p.bl = it.bl;
    p.last = it.bl == it.nbl - 1;
    const int row = it.blk * 16 + pr;
    const int c = it.col0 + pb * 16;
    const int cv = cols - c;
    const bool rok = row < rows;
    p.n = rok ? (cv < 0 ? 0 : (cv > 16 ? 16 : cv)) : 0;
    p.row = (rok && cv > 0) ? int64_t(it.s) * rows + row : -1;
    p.ptr = p.n ? static_cast<const void*>(src + int64_t(it.s) * a.seg_src + int64_t(row) * a.ld_src + c)
                : static_cast<const void*>(src);
    it.advance();
    return p;
  };

  StepPos p0 = pos_of();
  StepPos p1 = pos_of();
  uint4 r0[V], r1[V], r2[V];
  load_raw<T>(static_cast<const T*>(p0.ptr), p0.n, a.vec, r0);
  load_raw<T>(static_cast<const T*>(p1.ptr), p1.n, a.vec, r1);
  int buf = 0;

  auto step = [&](const StepPos& p, const uint4 (&raw)[V]) {
    uint8_t* tile = tiles + buf * 16 * kRow;
    // ---------------- phase 1: this thread's row piece
    if (GW) {
#pragma unroll
      for (int q = 0; q < V; ++q)
        *reinterpret_cast<uint4*>(tile + pr * kRow + chunk_off<T>(pb, q)) = raw[q];
    }
    if (GX && p.row >= 0) {
      float v[16];
      unpack16<T>(raw, v);
      fwht16_raw(v);
      if (MODE == kStats) {
#pragma unroll
        for (int i = 0; i < 16; ++i) sx.add(v[i]);
      } else {
        uint32_t c[16];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const uint2 cc = quant2<FAST_GX>(make_float2(v[i], v[i + 1]), qx);
          c[i] = cc.x; c[i + 1] = cc.y;
        }
        if (a.pack_gx) {
          uint32_t nb[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) nb[j] = (c[2 * j] & 0xFu) | ((c[2 * j + 1] & 0xFu) << 4);
          const uint2 out = make_uint2(pack_bytes(nb[0], nb[1], nb[2], nb[3]), pack_bytes(nb[4], nb[5], nb[6], nb[7]));
          *reinterpret_cast<uint2*>(a.dst_gx + p.row * a.ld_gx + ((p.col0 + pb * 16) >> 1)) = out;
        } else {
          uint4 out;
          out.x = pack_bytes(c[0], c[1], c[2], c[3]);
          out.y = pack_bytes(c[4], c[5], c[6], c[7]);
          out.z = pack_bytes(c[8], c[9], c[10], c[11]);
          out.w = pack_bytes(c[12], c[13], c[14], c[15]);
          *reinterpret_cast<uint4*>(a.dst_gx + p.row * a.ld_gx + p.col0 + pb * 16) = out;
        }
      }
    }
    if (!GW) return;
    __syncthreads();
    // ---------------- phase 2: columns (2t, 2t+1) of the tile, projection along rows
    if (tid < kTileCols / 2) {
      const int c = 2 * tid;
      const int64_t gc = p.col0 + c;
      if (gc < a.cols) {
        float2 pv[16];
        const int b = c >> 4, e = c & 15;
        if (sizeof(T) == 2) {
          const int off = chunk_off<T>(b, e >> 3) + 2 * (e & 7);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(tile + i * kRow + off);
            pv[i] = make_float2(bf_lo(w), bf_hi(w));
          }
        } else {
          const int off = chunk_off<T>(b, e >> 2) + 4 * (e & 3);
#pragma unroll
          for (int i = 0; i < 16; ++i) pv[i] = *reinterpret_cast<const float2*>(tile + i * kRow + off);
        }
        fwht16_pair(pv);
        const bool has2 = gc + 1 < a.cols;
        if (MODE == kStats) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if ((bitmap >> i) & 1u) {
              sw.add(pv[i].x);
              if (has2) sw.add(pv[i].y);
            }
          }
        } else {
          uint32_t wx[4] = {0, 0, 0, 0}, wy[4] = {0, 0, 0, 0};
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if ((bitmap >> i) & 1u) {
              const int j = BM ? __builtin_popcount(uint32_t(BM) & ((1u << i) - 1u))
                               : __popc(bitmap & ((1u << i) - 1u));
              const uint2 cc = quant2<FAST_GW>(pv[i], qw);
              const uint32_t bx = (cc.x & 0xFFu) << (8 * (j & 3));
              const uint32_t by = (cc.y & 0xFFu) << (8 * (j & 3));
              switch (j >> 2) {
                case 0: wx[0] |= bx; wy[0] |= by; break;
                case 1: wx[1] |= bx; wy[1] |= by; break;
                case 2: wx[2] |= bx; wy[2] |= by; break;
                default: wx[3] |= bx; wy[3] |= by; break;
              }
            }
          }
          uint8_t* ox = cbuf + c * cstride + p.bl * rank;
          uint8_t* oy = ox + cstride;
          if (rank == 16) {
            *reinterpret_cast<uint4*>(ox) = make_uint4(wx[0], wx[1], wx[2], wx[3]);
            *reinterpret_cast<uint4*>(oy) = make_uint4(wy[0], wy[1], wy[2], wy[3]);
          } else if (rank == 8) {
            *reinterpret_cast<uint2*>(ox) = make_uint2(wx[0], wx[1]);
            *reinterpret_cast<uint2*>(oy) = make_uint2(wy[0], wy[1]);
          } else if (rank == 4) {
            *reinterpret_cast<uint32_t*>(ox) = wx[0];
            *reinterpret_cast<uint32_t*>(oy) = wy[0];
          } else {
            for (int j = 0; j < rank; ++j) {
              ox[j] = uint8_t(wx[j >> 2] >> (8 * (j & 3)));
              oy[j] = uint8_t(wy[j >> 2] >> (8 * (j & 3)));
            }
          }
        }
      }
    }
    // ---------------- flush the work item's codes: (cols, K) K-major, >= 32B runs
    if (MODE == kQuant && p.last) {
      __syncthreads();
      const int run = p.nbl * rank;
      const int64_t k0 = p.gb0 * rank;
      const int ncols = int(a.cols - p.col0 < kTileCols ? a.cols - p.col0 : kTileCols);
      if ((run & 15) == 0 && (k0 & 15) == 0) {
        const int chunks = run >> 4;
        for (int i = tid; i < ncols * chunks; i += kThreads) {
          const int c = i / chunks, q = i - c * chunks;
          *reinterpret_cast<uint4*>(a.dst_gw + (p.col0 + c) * a.ld_gw + k0 + 16 * q) =
              *reinterpret_cast<const uint4*>(cbuf + c * cstride + 16 * q);
        }
      } else if ((run & 7) == 0 && (k0 & 7) == 0) {
        const int chunks = run >> 3;
        for (int i = tid; i < ncols * chunks; i += kThreads) {
          const int c = i / chunks, q = i - c * chunks;
          *reinterpret_cast<uint2*>(a.dst_gw + (p.col0 + c) * a.ld_gw + k0 + 8 * q) =
              *reinterpret_cast<const uint2*>(cbuf + c * cstride + 8 * q);
        }
      } else {
        for (int i = tid; i < ncols * run; i += kThreads) {
          const int c = i / run, q = i - c * run;
          a.dst_gw[(p.col0 + c) * a.ld_gw + k0 + q] = int8_t(cbuf[c * cstride + q]);
        }
      }
      __syncthreads();
    }
    buf ^= 1;
  };

  // software pipeline: loads run two steps ahead of the math
  while (p0.valid) {
    StepPos p2 = pos_of();
    load_raw<T>(static_cast<const T*>(p2.ptr), p2.n, a.vec, r2);
    step(p0, r0);
    if (!p1.valid) break;
    StepPos p3 = pos_of();
    load_raw<T>(static_cast<const T*>(p3.ptr), p3.n, a.vec, r0);
    step(p1, r1);
    if (!p2.valid) break;
    StepPos p4 = pos_of();
    load_raw<T>(static_cast<const T*>(p4.ptr), p4.n, a.vec, r1);
    step(p2, r2);
    p0 = p3;
    p1 = p4;
  }
}

template <typename T, int MODE, bool GX, bool GW, int BM>
__global__ void __launch_bounds__(kThreads) tile_kernel(TileArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  Stat sx, sw;
  if (MODE == kStats) {
    Quant dummy{};
    run_tile<BM, MODE, GX, GW, true, true, T>(a, dummy, dummy, smem, sx, sw);
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
    if (GX && qx.nonfinite && a.nonfinite) atomicOr(a.nonfinite, 1u);
    if (GW && qw.nonfinite && a.nonfinite) atomicOr(a.nonfinite, 1u);
  }
  const bool fx = !GX || qx.fast, fw = !GW || qw.fast;  // uniform across the grid
  if (fx && fw)
    run_tile<BM, MODE, GX, GW, true, true, T>(a, qx, qw, smem, sx, sw);
  else if (fx)
    run_tile<BM, MODE, GX, GW, true, false, T>(a, qx, qw, smem, sx, sw);
  else if (fw)
    run_tile<BM, MODE, GX, GW, false, true, T>(a, qx, qw, smem, sx, sw);
  else
    run_tile<BM, MODE, GX, GW, false, false, T>(a, qx, qw, smem, sx, sw);
}

template <typename T, int MODE, bool GX, bool GW, int BM>
void launch_tile(const TileArgs& a, cudaStream_t stream) {
  const int64_t ncol_tiles = (a.cols + kTileCols - 1) / kTileCols;
  const int64_t ngroups = (a.total_blocks + a.nb - 1) / a.nb;
  const int64_t items = ngroups * ncol_tiles;
  const int rank = GW ? a.rank : 0;
  const size_t smem = GW ? size_t(2 * 16 * Traits<T>::kRowBytes) + size_t(kTileCols) * (a.nb * rank + 16) : 0;
  static std::atomic<unsigned long long> attr{0};  // per template instance and device
  smem_attr_once(reinterpret_cast<const void*>(tile_kernel<T, MODE, GX, GW, BM>), 96 * 1024, attr);
  // persistent grid: exactly the resident CTAs, each walking several steps so
  // the register prefetch always has the next two blocks in flight
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_kernel<T, MODE, GX, GW, BM>,
                                                    kThreads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t cap = int64_t(num_sms()) * per_sm;
  const int grid = int(items < 1 ? 1 : (items > cap ? cap : items));
  tile_kernel<T, MODE, GX, GW, BM><<<grid, kThreads, smem, stream>>>(a);
}

template <typename T, int MODE, bool GX, bool GW>
void launch_bm(const TileArgs& a, cudaStream_t st) {
  if (!GW) return launch_tile<T, MODE, GX, GW, 0>(a, st);
  switch (a.bitmap) {
    case 0x5555: return launch_tile<T, MODE, GX, GW, 0x5555>(a, st);  // rank 8 (default plan)
    case 0x1111: return launch_tile<T, MODE, GX, GW, 0x1111>(a, st);  // rank 4
    case 0x0101: return launch_tile<T, MODE, GX, GW, 0x0101>(a, st);  // rank 2
    case 0xFFFF: return launch_tile<T, MODE, GX, GW, 0xFFFF>(a, st);  // full (H.W, rank 16)
    default: return launch_tile<T, MODE, GX, GW, 0>(a, st);           // calibrated bases
  }
}

template <typename T>
void launch_modes(const TileArgs& a, int mode, bool gx, bool gw, cudaStream_t st) {
  if (mode == kStats) {
    if (gx && gw) launch_bm<T, kStats, true, true>(a, st);
    else if (gx) launch_bm<T, kStats, true, false>(a, st);
    else launch_bm<T, kStats, false, true>(a, st);
  } else {
    if (gx && gw) launch_bm<T, kQuant, true, true>(a, st);
    else if (gx) launch_bm<T, kQuant, true, false>(a, st);
    else launch_bm<T, kQuant, false, true>(a, st);
  }
}

// Blocks per work item: >= 32-byte output runs per column when the problem is
// large, while keeping >= ~3 work items per SM.
int choose_nb(int64_t total_blocks, int64_t cols, int rank) {
  int nb = rank >= 8 ? 4 : (rank >= 4 ? 8 : 16);
  const int64_t ncol_tiles = (cols + kTileCols - 1) / kTileCols;
  while (nb > 1 && ((total_blocks + nb - 1) / nb) * ncol_tiles < int64_t(num_sms()) * 3) nb >>= 1;
  return nb;
}

}  // namespace

void launch_transform_fallback(const TransformArgs& t, int mode, cudaStream_t stream) {
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
  a.nonfinite = nonfinite_word();
  a.pack_gx = t.pack_gx;
  const size_t esz = t.dtype == kBF16 ? 2 : 4;
  a.vec = (reinterpret_cast<uintptr_t>(t.src) % 16 == 0) && ((t.ld_src * esz) % 16 == 0) &&
          ((t.seg_src * esz) % 16 == 0);
  a.nb = t.do_gw ? choose_nb(a.total_blocks, t.cols, a.rank) : 4;
  if (t.dtype == kBF16)
    launch_modes<__nv_bfloat16>(a, mode, t.do_gx, t.do_gw, stream);
  else
    launch_modes<float>(a, mode, t.do_gx, t.do_gw, stream);
}

}  // namespace hlq
