// Device helpers shared by the transform kernels: packed fp32x2 arithmetic,
// the 16-point Walsh-Hadamard butterflies, transformed-value statistics and
// the bit-exact pseudo-stochastic quantizer (see hlq_transform.cu header for
// the exactness argument).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace hlq {
namespace dev {

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: ulp 1, small integers in the low mantissa bits

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
__device__ __forceinline__ float2 f2sub_rp(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rp.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2fma_rp(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rp.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// bf16 -> fp32: both halves on the ALU pipe (PRMT / LOP3), keeping the FMA
// pipe for the butterflies and the quantizer
__device__ __forceinline__ float bf_lo(uint32_t w) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(r) : "r"(w));
  return __uint_as_float(r);
}
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// ------------------------------------------------------------------ transforms
// Un-normalised 16-point FWHT of one vector (the 0.25 is folded into the
// quantizer divisor).  Register pairs (v[i], v[i+8]) run stages h = 1, 2, 4
// as f32x2; stage 8 pairs the two lanes of each register pair.  Stage order
// h = 1, 2, 4, 8 is the reference's (hadamard.py:125-133).
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

// Two independent vectors at once (lane x and lane y of each float2).  The
// compiler drops butterflies whose outputs are never read (pruned projection).
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
// Per-thread statistics of transformed values, two values per update, all on
// 3-input FMNMX with |.| operand modifiers:
//   amax  max |w| with NaN propagation (a NaN/Inf input surfaces as bits
//         >= 0x7F800000);
//   mnz   min over nonzero |w| of the float whose bits are bits(|w|) - 1: the
//         decrement (an IMAD, FMA pipe) turns +-0 into a NaN pattern that the
//         NaN-ignoring min skips, and is monotone on nonzero magnitudes.
struct Stat {
  float amax = 0.0f;
  float mnz = __builtin_huge_valf();  // +inf: no nonzero value seen
  __device__ __forceinline__ static float dec(float a) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(__float_as_uint(a)), "r"(1u), "r"(0xFFFFFFFFu));
    return __uint_as_float(r);
  }
  __device__ __forceinline__ void add2(float a, float b) {
    asm("{.reg .f32 t0, t1;\n\tabs.f32 t0, %1;\n\tabs.f32 t1, %2;\n\t"
        "max.NaN.f32 %0, %0, t0, t1;}" : "+f"(amax) : "f"(a), "f"(b));
    asm("{.reg .f32 t0, t1;\n\tabs.f32 t0, %1;\n\tabs.f32 t1, %2;\n\t"
        "min.f32 %0, %0, t0, t1;}" : "+f"(mnz) : "f"(dec(a)), "f"(dec(b)));
  }
  __device__ __forceinline__ void add(float a) { add2(a, 0.0f); }
  // amax only (the bound-test STATS pass takes min nonzero from the inputs)
  __device__ __forceinline__ void amax2(float a, float b) {
    asm("{.reg .f32 t0, t1;\n\tabs.f32 t0, %1;\n\tabs.f32 t1, %2;\n\t"
        "max.NaN.f32 %0, %0, t0, t1;}" : "+f"(amax) : "f"(a), "f"(b));
  }
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float oa = __shfl_xor_sync(0xffffffffu, amax, o);
      asm("max.NaN.f32 %0, %0, %1;" : "+f"(amax) : "f"(oa));
      const float om = __shfl_xor_sync(0xffffffffu, mnz, o);
      asm("min.f32 %0, %0, %1;" : "+f"(mnz) : "f"(om));
    }
  }
  // global layout {amax bits, ~(minnz bits - 1)}, both max-reduced so a zero
  // memset is the identity (NaN from max.NaN is 0x7FFFFFFF: flagged non-finite)
  // Fire-and-forget reductions (RED, no returned value): the committing thread
  // does not wait for an L2 round trip per word before it arrives at the grid
  // barrier, whose release orders them.
  __device__ __forceinline__ void commit(uint32_t* g) const {
    const uint32_t ab = __float_as_uint(amax) & 0x7FFFFFFFu;
    if (ab) asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(g), "r"(ab) : "memory");
    const uint32_t mb = __float_as_uint(mnz);
    if (mb < 0x7F800000u) asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(g + 1), "r"(~mb) : "memory");
  }
};

// ------------------------------------------------------------------ bound statistics (bf16 sources)
// The STATS pass needs max |w| over the transformed values exactly, but a block
// can only raise the running maximum if its L1 norm can reach it: every
// butterfly output satisfies |RN(a +- b)| <= RN(|a| + |b|) (RN is monotone),
// so by induction each computed output of a block is <= the fp32 pairwise
// tree sum of the block's |x|, which is <= L1 * (1 + 2^-24)^4.  The test sums
// the |x| words as bf16x2 (4 tree levels, each RN step loses at most a factor
// (1 - 2^-8)): a block whose bf16 sum is <= RD(0.96875 * m) for an exact
// running maximum m of other blocks has every output < m and is skipped; the
// others run the exact fp32 butterflies.  NaN / Inf sums never pass the test.
//
// Min nonzero guard of the fast division (make_quant), from the INPUTS: every
// bf16 value is a multiple of g = 2^(E_min - 7) (E_min the exponent of the
// smallest nonzero |x|, -126 for subnormals), so is every fp32 butterfly
// output (an inexact RN result is a multiple of its ulp, itself >= g), hence
// a nonzero |w| >= g >= min|x| * 2^-8.  The minimum runs on s16x2 lanes of
// (|x| bits + 0x7FFF): 0 maps to 0x7FFF (the s16 maximum, never selected
// while a nonzero lane exists), |x| bits a >= 1 to -32769 + a (monotone).
__device__ __forceinline__ uint32_t bf2_add(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t s16x2_min3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("min.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));  // ptxas fuses the pair into VIMNMX3
  asm("min.s16x2 %0, %0, %1;" : "+r"(d) : "r"(c));
  return d;
}
constexpr uint32_t kAbs2 = 0x7FFF7FFFu;
// Pairwise bf16x2 tree over n |x| words (n = 8 or 16, 3 / 4 levels).
template <int N>
__device__ __forceinline__ uint32_t bf2_tree(const uint32_t (&a)[N]) {
  uint32_t t[N / 2];
#pragma unroll
  for (int i = 0; i < N / 2; ++i) t[i] = bf2_add(a[2 * i], a[2 * i + 1]);
#pragma unroll
  for (int h = N / 4; h >= 1; h >>= 1)
#pragma unroll
    for (int i = 0; i < h; ++i) t[i] = bf2_add(t[2 * i], t[2 * i + 1]);
  return t[0];
}
// skip threshold from an exact running maximum (0: only all-zero blocks skip;
// tiny maxima never skip, so subnormal bf16 sums stay inside the margin)
__device__ __forceinline__ float bound_thr(float m) {
  return m >= 0x1p-100f ? __fmul_rd(m, 0.96875f) : 0.0f;
}
// the two bf16 lanes as fp32 and their NaN-propagating max
__device__ __forceinline__ float bf2_lane_max(uint32_t s) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(__uint_as_float(s << 16)), "f"(__uint_as_float(s & 0xFFFF0000u)));
  return r;
}
// running s16x2 minimum -> the Stat::mnz encoding (bits - 1 of the lower bound
// min|x| * 2^-8 of every nonzero transformed |w|); +inf when no nonzero input
__device__ __forceinline__ float mz_to_mnz(uint32_t mz) {
  const int lo = int(int16_t(mz & 0xFFFFu)), hi = int(int16_t(mz >> 16));
  const int v = lo < hi ? lo : hi;
  if (v == 0x7FFF) return __builtin_huge_valf();
  const uint32_t a = uint32_t(v + 32769);                 // |x| bf16 bits of the smallest nonzero input
  const float lb = __fmul_rn(__uint_as_float(a << 16), 0x1p-8f);  // exact (8 significant bits)
  return __uint_as_float(__float_as_uint(lb) - 1u);
}

// ------------------------------------------------------------------ quantizer
struct Quant {
  float s, d, r, lim, qmax;
  uint32_t lim16;   // (qmax, qmax) as s16x2
  uint32_t nlim16;  // (-qmax, -qmax) as s16x2
  bool fast;
  bool nonfinite;  // the operand's amax bits were NaN / Inf
};

// OR the operand's non-finite status into the device's sticky flag (one thread per operand)
__device__ __forceinline__ void flag_nonfinite(const Quant& q, uint32_t* word) {
  if (q.nonfinite && word) atomicOr(word, 1u);
}

// scale = f32(amax_v) / f32(qmax), 0 -> 1 (quantize.py:94-100), amax_v = RN(0.25 * max|w|)
// (= max|RN(0.25 w)| because rounding is monotone).
__device__ __forceinline__ Quant make_quant(const uint32_t* g, int bits) {
  Quant q;
  const int qm = (1 << (bits - 1)) - 1;
  q.qmax = float(qm);
  q.lim16 = (uint32_t(qm) & 0xFFFFu) * 0x10001u;
  q.nlim16 = (uint32_t(-qm) & 0xFFFFu) * 0x10001u;
  // L1-bypassing loads: in the fused kernel these words were written by other
  // CTAs' atomics just before the grid barrier
  const uint32_t g0 = __ldcg(g), g1 = __ldcg(g + 1);
  q.nonfinite = g0 >= 0x7F800000u;
  const float amax_w = __uint_as_float(g0);
  const float amax_v = __fmul_rn(amax_w, 0.25f);
  float s = __fdiv_rn(amax_v, q.qmax);
  if (s == 0.0f) s = 1.0f;
  q.s = s;
  q.d = __fmul_rn(s, 1.0f / 512.0f);
  q.r = __frcp_rn(q.d);
  q.lim = 2048.0f * q.qmax;
  const uint32_t inv = g1;
  const float minnz = inv ? __uint_as_float(~inv + 1u) : 0.0f;  // 0: no nonzero value at all
  q.fast = (g0 < 0x7F800000u) && s > 0x1p-116f &&
           (minnz == 0.0f || (minnz >= 0x1p-100f && minnz >= __fmul_rn(s, 0x1p-108f)));
  return q;
}

// The reference rounds up iff RN(q - floor(q)) * 2048 > u (quantize.py:143-144).
// q - floor(q) is exact except for q in (-0.5, 0), where it is RN(q + 1): in
// the scaled domain (Q = 2048 q) the test is RN(Q + 2048) > u, i.e. (u integer,
// ties to even) Q + 2048 > u + 2^-14 -- so those lanes use Qr = RU(Q - 2^-14)
// (RU keeps the comparison with every integer boundary), all others Qr = Q.
// RU(Q - 2^-14) == Q for Q <= -1024 (ulp >= 2^-13), and as int32 bit patterns
// RU(Q - 2^-14) > Q exactly when Q < 0 (larger magnitude, sign set) while for
// Q >= 0 it is below Q: one integer max selects Qr.  (Found by the batch-128
// ViT qkv parity test: 1 of 58 M codes had Q + 2048 - u in (0, 2^-14].)
__device__ __forceinline__ float2 ref_frac_adjust(float2 Q) {
  const float2 t = f2add_rp(Q, f2(-0x1p-14f));
  return make_float2(__int_as_float(max(__float_as_int(Q.x), __float_as_int(t.x))),
                     __int_as_float(max(__float_as_int(Q.y), __float_as_int(t.y))));
}

// Unclamped codes of two values as two s16 lanes: code = ceil((Qr - u) / 2048),
// Qr = ref_frac_adjust(Q), Q = RN(w / d) by reciprocal-FMA division, u = bits(w) & 0x7FF.
//   U  = 2^23 + u as a float (one LOP3: OR the draw into 2^23's mantissa);
//   z  = RU(Q - U) = RU(y - 2^23), y = Q - u in (-2^19, 2^19): a grid of
//        spacing <= 1 around -2^23, so z + 2^23 = g is the smallest grid point
//        >= y, and ceil(g / 2048) = ceil(y / 2048) (multiples of 2048 lie on
//        the grid);
//   c  = RU(z * 2^-11 + (M + 4096)) = M + ceil(g / 2048), M = 1.5 * 2^23 (ulp 1):
//        the low bits of c are the two's-complement code.
__device__ __forceinline__ uint32_t quant_fast2(float2 w, const Quant& q) {
  const float2 Q0 = f2mul(w, f2(q.r));
  const float2 e = f2fma(Q0, f2(-q.d), w);
  const float2 Q = ref_frac_adjust(f2fma(e, f2(q.r), Q0));
  uint32_t ux, uy;
  const uint32_t magic = 0x4B000000u;  // 2^23
  asm("lop3.b32 %0, %1, 0x7FF, %2, 0xEA;" : "=r"(ux) : "r"(__float_as_uint(w.x)), "r"(magic));
  asm("lop3.b32 %0, %1, 0x7FF, %2, 0xEA;" : "=r"(uy) : "r"(__float_as_uint(w.y)), "r"(magic));
  const float2 z = f2sub_rp(Q, make_float2(__uint_as_float(ux), __uint_as_float(uy)));  // RU(Q - U)
  const float2 c = f2fma_rp(z, f2(1.0f / 2048.0f), f2(kMagic + 4096.0f));
  return __byte_perm(__float_as_uint(c.x), __float_as_uint(c.y), 0x5410);
}

// Literal restatement of quantize.py:140-145 (IEEE division), used when the
// fast path's guard fails for the tensor.  Returns the clamped code.
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

// Clip to +-qmax.  Only the upper bound can bind: |q| = |v/s| <= qmax*(1 + 2^-23)
// (s = RN(amax/qmax)), so a code below -qmax would need frac*2048 <= u with
// frac >= 1 - 2^-20, impossible for u <= 2047; above, q = qmax + tiny rounds
// up to qmax + 1 when u == 0.
__device__ __forceinline__ uint32_t clamp_s16x2(uint32_t p, const Quant& q) {
  uint32_t r;
  asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(p), "r"(q.lim16));
  return r;
}

// Two clamped codes as s16x2.
template <bool FAST>
__device__ __forceinline__ uint32_t quant2(float2 w, const Quant& q) {
  if (FAST) return clamp_s16x2(quant_fast2(w, q), q);
  return (uint32_t(quant_exact(w.x, q)) & 0xFFFFu) | (uint32_t(quant_exact(w.y, q)) << 16);
}

// Four codes (two s16x2 words) -> four int8 bytes.
__device__ __forceinline__ uint32_t pack4(uint32_t p01, uint32_t p23) {
  return __byte_perm(p01, p23, 0x6420);
}

}  // namespace dev
}  // namespace hlq
