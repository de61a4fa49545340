// Integer GEMM with fused dequantization for both HLQ products:
//
//   dX  = deq( Q4(H.gy) [T x O_p]  . Q4(H.W)^T [I x O_p]^T )          (backprop.py:367-369)
//   dW  = deq( Q8(P.gy)^T [O x K]  . Q8(P.X)^T  [I x K]^T ) * extra   (backprop.py:407-410)
//
// Both operands are int8 codes stored K-major (row = M or N index, K contiguous),
// so the same kernel serves both products:  D[m, n] = sum_k A[m, k] * B[n, k].
//
// sm_100a structure (one persistent CTA per SM, 8 warps):
//   warp 0      TMA producer: 128x128 A tile + BNx128 B tile per stage (SWIZZLE_128B)
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::i8, M=128, N=BN, K=32 per op,
//               int32 accumulators in TMEM, two accumulator buffers (2*BN columns)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> registers -> dequant -> global
// Exact epilogue (quantize.py:181-187): out = f32( f64(acc) * (f64(f32(sa*sb)) * extra) ).
// Fast epilogue (training): out = f32(acc) * f32(sa*sb*extra), fp32 or bf16 output.
// int32 accumulation is exact while K * qmax_a * qmax_b < 2^31 (checked by the caller).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <algorithm>
#include <cstring>
#include <vector>

#include "hlq_internal.h"
#include "hlq_ptx.cuh"

namespace hlq {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 128;  // bytes of K per stage = one 128B swizzle row
constexpr int kThreads = 256;
// single-CTA int8-A kernel: two epilogue warps per TMEM lane quarter (warps 4-7
// and 8-11) splitting each tile's columns -- one warp per SMSP could not keep up
// with the MMAs (fc2 dX: the MMA warp waited on TMEM-empty, tensor pipe 54 %)
constexpr int kThreadsE2 = 384;
// Packed int4 A operand: + kConvWarps converter warps (8 .. 8 + kConvWarps - 1)
constexpr int kConvWarps = 8;
constexpr int kConvThreads = 32 * kConvWarps;
constexpr int kThreadsA4 = 256 + kConvThreads;
constexpr uint32_t kPackedA = kBM * kBK / 2;  // one stage of packed A: 128 rows x 64 bytes

// ---------------------------------------------------------------- packed int4 A
// The gx codes Q4(H.gy) can live in HBM packed two per byte, low nibble first
// (the ACBP container's nibble order, acbp.py:56-61) -- half the bytes of the
// int8 form.  tcgen05 has no int4 MMA and TMA cannot widen nibbles, so the TMA
// loads each 128 x 64-byte packed tile into the UPPER half of the stage's A
// slot and 4 converter warps widen it in place into the 128 x 128-byte
// SWIZZLE_128B K-major int8 tile kind::i8 reads (all packed input is read into
// registers, then a named barrier, then the writes).  A nibble placed in the
// HIGH half of its byte is the int8 value 16 * code (two's complement), so the
// widening needs no sign extension: the MMA accumulates 16 * sum(a b) (exact:
// 16 * 49 * K < 2^31 for K < 2.7 M) and the host folds 1/16 into the dequant
// scale -- power-of-two scalings are exact, so the outputs are bit-identical.
__device__ __forceinline__ void unpack8(uint32_t x, uint32_t& o0, uint32_t& o1) {
  const uint32_t lo = (x << 4) & 0xF0F0F0F0u;  // 16 * codes 0, 2, 4, 6
  const uint32_t hi = x & 0xF0F0F0F0u;         // 16 * codes 1, 3, 5, 7
  o0 = __byte_perm(lo, hi, 0x5140);
  o1 = __byte_perm(lo, hi, 0x7362);
}
// ct = converter thread 0 .. kConvThreads-1.  Unit u = (row u / 4, 16 packed
// bytes u % 4 = K codes [32 q, 32 q + 32)) -> int8 chunks 2q and 2q+1 of the
// row, at chunk position c ^ (row % 8) (the 128B swizzle of a 1024-byte
// aligned tile).
__device__ __forceinline__ void convert_a4(uint8_t* slot, int ct) {
  constexpr int kUnits = 512 / kConvThreads;
  const uint32_t base = ptx::smem_u32(slot);
  uint4 in[kUnits];
#pragma unroll
  for (int j = 0; j < kUnits; ++j) in[j] = ptx::lds128(base + kPackedA + uint32_t(ct + kConvThreads * j) * 16u);
  asm volatile("bar.sync 3, %0;" ::"n"(kConvThreads) : "memory");
#pragma unroll
  for (int j = 0; j < kUnits; ++j) {
    const int u = ct + kConvThreads * j, r = u >> 2, q = u & 3;
    uint32_t o[8];
    unpack8(in[j].x, o[0], o[1]);
    unpack8(in[j].y, o[2], o[3]);
    unpack8(in[j].z, o[4], o[5]);
    unpack8(in[j].w, o[6], o[7]);
    const uint32_t row = base + uint32_t(r) * 128u;
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((uint32_t(2 * q) ^ (r & 7)) << 4)),
                 "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]) : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((uint32_t(2 * q + 1) ^ (r & 7)) << 4)),
                 "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]) : "memory");
  }
  ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
}

template <int BN, int STAGES>
struct GemmCfg;

// Per-warp staging for the TMA-store epilogue: 2 buffers x 32 rows x 128 B.
constexpr uint32_t kStgBytes = 2 * 32 * 128;
constexpr uint32_t kStgAll = 4 * kStgBytes;

// Fast epilogue of one 32 x 32 chunk (this warp's 32 TMEM lanes = rows) through
// shared memory and one TMA tile store: rows are written swizzled (SW64 for
// bf16 / SW128 for fp32, matching the store map) so the row-per-thread 16-byte
// writes are bank-conflict free; TMA clips rows / columns outside the output.
__device__ __forceinline__ void store_chunk_tma(const uint32_t (&acc)[32], float fscale, int out_dtype,
                                                uint8_t* buf, uint32_t lane, const CUtensorMap* map_o,
                                                int32_t col0, int32_t row0) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(__int2float_rn(int(acc[j])), fscale);
  if (out_dtype == kBF16) {
    uint8_t* rowp = buf + lane * 64;
    const uint32_t sw = (lane >> 1) & 3;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 t = __floats2bfloat162_rn(v[8 * q + 2 * k], v[8 * q + 2 * k + 1]);
        w[k] = *reinterpret_cast<uint32_t*>(&t);
      }
      *reinterpret_cast<uint4*>(rowp + 16 * (q ^ sw)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
    uint8_t* rowp = buf + lane * 128;
    const uint32_t sw = lane & 7;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(rowp + 16 * (q ^ sw)) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  ptx::fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    ptx::tma_store_2d(map_o, buf, col0, row0);
    ptx::bulk_commit();
  }
}

// bf16 fast epilogue of two adjacent 32 x 32 chunks as ONE 32 x 64 tile store:
// 128-byte rows (SW128, conflict-free row-per-thread 16-byte writes).  The
// 64-byte rows of single-chunk bf16 stores held the TMA store path to ~4 TB/s
// (fc2 dX: the output write, not the tensor pipe, set the kernel time).
__device__ __forceinline__ void store_pair_tma_bf16(const uint32_t (&a0)[32], const uint32_t (&a1)[32], float fscale,
                                                    uint8_t* buf, uint32_t lane, const CUtensorMap* map_o,
                                                    int32_t col0, int32_t row0) {
  uint8_t* rowp = buf + lane * 128;
  const uint32_t sw = lane & 7;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t(&a)[32] = q < 4 ? a0 : a1;
    const int j0 = 8 * (q & 3);
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float x = __fmul_rn(__int2float_rn(int(a[j0 + 2 * k])), fscale);
      const float y = __fmul_rn(__int2float_rn(int(a[j0 + 2 * k + 1])), fscale);
      __nv_bfloat162 t = __floats2bfloat162_rn(x, y);
      w[k] = *reinterpret_cast<uint32_t*>(&t);
    }
    *reinterpret_cast<uint4*>(rowp + 16 * (q ^ sw)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  ptx::fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    ptx::tma_store_2d(map_o, buf, col0, row0);
    ptx::bulk_commit();
  }
}

template <int BN, int STAGES>
struct GemmCfg {
  static constexpr uint32_t kABytes = kBM * kBK;
  static constexpr uint32_t kBBytes = BN * kBK;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kTmemCols = 2 * BN;  // 256 or 512: power of two
  static constexpr size_t kSmem = size_t(STAGES) * kStageBytes + kStgAll + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ void store_row_chunk(const uint32_t (&acc)[32], int64_t row, int64_t col0,
                                                int64_t N, int epilogue, double dscale, float fscale,
                                                void* out, int out_dtype, int64_t ldo, bool vec_ok,
                                                int32_t* acc_out, int64_t ld_acc) {
  const int64_t nvalid = N - col0;
  if (acc_out) {
    int32_t* a = acc_out + row * ld_acc + col0;
    if (nvalid >= 32 && (ld_acc % 4 == 0) && ((reinterpret_cast<uintptr_t>(acc_out) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<int4*>(a + j) =
            make_int4(int(acc[j]), int(acc[j + 1]), int(acc[j + 2]), int(acc[j + 3]));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) a[j] = int(acc[j]);
    }
  }
  if (!out) return;
  float v[32];
  if (epilogue == kEpiExact) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __double2float_rn(__dmul_rn(double(int(acc[j])), dscale));
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(__int2float_rn(int(acc[j])), fscale);
  }
  if (out_dtype == kF32) {
    float* o = static_cast<float*>(out) + row * ldo + col0;
    if (nvalid >= 32 && vec_ok) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) o[j] = v[j];
    }
  } else {
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out) + row * ldo + col0;
    if (nvalid >= 32 && vec_ok) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 p;
        __nv_bfloat162 t0 = __floats2bfloat162_rn(v[j], v[j + 1]);
        __nv_bfloat162 t1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
        __nv_bfloat162 t2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
        __nv_bfloat162 t3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
        p.x = *reinterpret_cast<uint32_t*>(&t0);
        p.y = *reinterpret_cast<uint32_t*>(&t1);
        p.z = *reinterpret_cast<uint32_t*>(&t2);
        p.w = *reinterpret_cast<uint32_t*>(&t3);
        *reinterpret_cast<uint4*>(o + j) = p;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) o[j] = __float2bfloat16_rn(v[j]);
    }
  }
}

// Split-K (dW: few output tiles, very long K): work unit u = tile * splits + split
// covers K blocks [split*nk/splits, (split+1)*nk/splits) and stores its int32
// partial tile to workspace slab `split`; splitk_finalize then sums the slabs
// (integers: exact in any order) and runs the same dequant epilogue.
// Implicit-GEMM conv dgrad: A[m, (tap, o)] = G codes at output pixel m shifted
// by the flipped tap, read by im2col-mode TMA (zero padding from the map's
// bounding box); B[c, (tap, o)] = W codes of the tap, a 4-D tiled map
// (o, tap_j, tap_i, c).  K loop = taps x channel chunks of 128.
// Stride s > 1 runs as s^2 output phases (h = s h' + ph, w = s w' + pw): phase
// (ph, pw) is a stride-1 correlation of G with the taps i = i0 + s t
// (i0 = (ph + pad) mod s), G row h' + (ph + pad - i0)/s - t -- no zero-inserted
// G and no dcols tensor; its rows are scattered to dX by the epilogue.
struct ConvGeo {
  int conv;        // 0: plain GEMM
  int Ho, Wo;      // the output grid this launch walks (a phase grid for s > 1)
  int kh, kw;      // taps of this phase along h / w
  int lo_h, lo_w;  // im2col base offset of the flipped-tap traversal (-(k-1-pad) at stride 1)
  int nkc;         // 128-byte channel chunks per tap
  int s, ph, pw;   // output remap: row (b, h', w') -> dX pixel (b, s h' + ph, s w' + pw)
  int H, W;        // dX spatial extent
};

template <int BN, int STAGES, bool A4>
__global__ void __launch_bounds__(A4 ? kThreadsA4 : kThreadsE2, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_o, int tma_out,
                   int M, int N, int K, int groups, const float* __restrict__ sa, const float* __restrict__ sb,
                   double extra, int epilogue, void* out, int out_dtype, int64_t ldo,
                   int32_t* acc_out, int64_t ld_acc, int splits, int32_t* __restrict__ slabs,
                   const ConvGeo geo) {
  using Cfg = GemmCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::kABytes;
  uint8_t* stg = sB + STAGES * Cfg::kBBytes;  // 1024-aligned: stage bytes are multiples of 1 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + kStgAll);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* aready = tempty + 2;  // A4: the stage's A tile is converted (4 converter warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aready + STAGES);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&map_a);
    ptx::tma_prefetch_desc(&map_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&aready[s], kConvWarps);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], A4 ? 128 : 256);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, Cfg::kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel's tail; its outputs (codes, scales) are read only from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const int num_m = (M + kBM - 1) / kBM;
  const int num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int units = tiles * splits;
  const int nk_g = (K + kBK - 1) / kBK;  // K blocks per group
  const int nk = geo.conv ? geo.kh * geo.kw * geo.nkc : nk_g * groups;  // groups / taps accumulate

  if (warp == 0) {
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int t = u / splits, sp = u - t * splits;
        const int mb = t / num_n, nb = t - mb * num_n;
        const int kb0 = int(int64_t(sp) * nk / splits), kb1 = int(int64_t(sp + 1) * nk / splits);
        int g = kb0 / nk_g, kg = kb0 - g * nk_g;
        // conv: first output pixel of this M tile, as im2col box coordinates
        int pw = 0, ph = 0, pn = 0;
        if (geo.conv) {
          const int p0 = mb * kBM, hw = geo.Ho * geo.Wo;
          pn = p0 / hw;
          const int rem = p0 - pn * hw;
          ph = rem / geo.Wo;
          pw = rem - ph * geo.Wo;
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait_sleep(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], A4 ? kPackedA + Cfg::kBBytes : Cfg::kStageBytes);
          if (A4) {
            // packed A (64 bytes of K per row) into the upper half of the A slot
            ptx::tma_load_3d(sA + stage * Cfg::kABytes + kPackedA, &map_a, &full[stage], kg * (kBK / 2), mb * kBM,
                             g);
            ptx::tma_load_3d(sB + stage * Cfg::kBBytes, &map_b, &full[stage], kg * kBK, nb * BN, g);
          } else if (geo.conv) {
            const int tap = kb / geo.nkc, oc = kb - tap * geo.nkc;
            const int ti = tap / geo.kw, tj = tap - ti * geo.kw;
            // flipped tap: dX[h, w] += G[h + pad - i, w + pad - j] W[i, j] (per phase: t = tap index)
            ptx::tma_load_im2col_4d(sA + stage * Cfg::kABytes, &map_a, &full[stage], oc * kBK, pw + geo.lo_w,
                                    ph + geo.lo_h, pn, uint16_t(geo.kw - 1 - tj), uint16_t(geo.kh - 1 - ti));
            ptx::tma_load_4d(sB + stage * Cfg::kBBytes, &map_b, &full[stage], oc * kBK, tj, ti, nb * BN);
          } else {
            ptx::tma_load_3d(sA + stage * Cfg::kABytes, &map_a, &full[stage], kg * kBK, mb * kBM, g);
            ptx::tma_load_3d(sB + stage * Cfg::kBBytes, &map_b, &full[stage], kg * kBK, nb * BN, g);
          }
          if (++kg == nk_g) { kg = 0; ++g; }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = ptx::idesc_i8(kBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int sp = u % splits;
      const int kb0 = int(int64_t(sp) * nk / splits), kb1 = int(int64_t(sp + 1) * nk / splits);
      ptx::mbar_wait_sleep(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
      for (int kb = kb0; kb < kb1; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        if (A4) ptx::mbar_wait(&aready[stage], phase);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint64_t a_desc = ptx::desc_kmajor_sw128(ptx::smem_u32(sA + stage * Cfg::kABytes));
          const uint64_t b_desc = ptx::desc_kmajor_sw128(ptx::smem_u32(sB + stage * Cfg::kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k) {
            // advance the start address by 32 bytes of K inside the swizzle atom
            ptx::mma_i8(d_tmem, a_desc + uint64_t((k * 32) >> 4), b_desc + uint64_t((k * 32) >> 4),
                        idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          ptx::mma_commit(&empty[stage]);
          if (kb == kb1 - 1) ptx::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (A4 && warp >= 8) {
    // converters: the same (unit, K block) walk as the MMA issuer
    const int ct = int(threadIdx.x) - 256;
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int sp = u % splits;
      const int kb0 = int(int64_t(sp) * nk / splits), kb1 = int(int64_t(sp + 1) * nk / splits);
      for (int kb = kb0; kb < kb1; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        convert_a4(sA + stage * Cfg::kABytes, ct);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&aready[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if ((warp >= 4 && warp < 8) || (!A4 && warp >= 8 && warp < 12)) {
    const uint32_t quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
    constexpr int kGroups = A4 ? 1 : 2;  // epilogue warps per quarter: chunk c belongs to group c % kGroups
    const int grp = warp >= 8 ? 1 : 0;
    const float comb = __fmul_rn(*sa, *sb);
    const double dscale = __dmul_rn(double(comb), extra);
    const float fscale = float(dscale);
    const bool vec_ok = (ldo % 8 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int t = u / splits, sp = u - t * splits;
      const int mb = t / num_n, nb = t - mb * num_n;
      ptx::mbar_wait_sleep(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int rl = quarter * 32 + lane;  // row inside the tile
      const int64_t row = int64_t(mb) * kBM + rl;
      if (splits == 1 && tma_out) {
        // staging: A4 -- 2 buffers of 4 KB per warp (warps 4-7); otherwise one 4 KB
        // buffer per warp (warps 4-11), the other warp of the quarter hides the wait
        uint8_t* wbuf = A4 ? stg + quarter * kStgBytes : stg + (quarter + 4 * grp) * (kStgBytes / 2);
        const int32_t row0 = mb * kBM + int32_t(quarter) * 32;
        if (out_dtype == kBF16) {
#pragma unroll 1
          for (int c = 2 * grp; c < BN / 32; c += 2 * kGroups) {  // 32 x 64 tiles (128-byte rows)
            const int32_t col0 = nb * BN + c * 32;
            uint32_t r0[32], r1[32];
            ptx::tmem_ld_32x32b_x32(tmem_base + ((quarter * 32) << 16) + uint32_t(acc * BN + c * 32), r0);
            ptx::tmem_ld_32x32b_x32(tmem_base + ((quarter * 32) << 16) + uint32_t(acc * BN + c * 32 + 32), r1);
            ptx::tmem_ld_wait();
            if (lane == 0) {  // the store that last used this buffer has read it
              if (A4) ptx::bulk_wait_read<1>(); else ptx::bulk_wait_read<0>();
            }
            __syncwarp();
            if (row0 < M && col0 < N)
              store_pair_tma_bf16(r0, r1, fscale, A4 ? wbuf + ((c >> 1) & 1) * (kStgBytes / 2) : wbuf, lane, &map_o,
                                  col0, row0);
          }
        } else {
#pragma unroll 1
        for (int c = grp; c < BN / 32; c += kGroups) {
          const int32_t col0 = nb * BN + c * 32;
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(tmem_base + ((quarter * 32) << 16) + uint32_t(acc * BN + c * 32), r);
          ptx::tmem_ld_wait();
          if (lane == 0) {
            if (A4) ptx::bulk_wait_read<1>(); else ptx::bulk_wait_read<0>();
          }
          __syncwarp();
          if (row0 < M && col0 < N)
            store_chunk_tma(r, fscale, out_dtype, A4 ? wbuf + (c & 1) * (kStgBytes / 2) : wbuf, lane, &map_o, col0,
                            row0);
        }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
      } else if (splits == 1) {
#pragma unroll 1
        for (int c = grp; c < BN / 32; c += kGroups) {
          const int64_t col0 = int64_t(nb) * BN + c * 32;
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(tmem_base + ((quarter * 32) << 16) + uint32_t(acc * BN + c * 32), r);
          ptx::tmem_ld_wait();
          if (row < M && col0 < N) {
            int64_t orow = row;
            if (geo.conv && geo.s > 1) {  // phase row (b, h', w') -> dX pixel (b, s h' + ph, s w' + pw)
              const int64_t hw = int64_t(geo.Ho) * geo.Wo;
              const int64_t b = row / hw, r2 = row - b * hw, hp = r2 / geo.Wo, wp = r2 - hp * geo.Wo;
              orow = (b * geo.H + geo.s * hp + geo.ph) * geo.W + geo.s * wp + geo.pw;
            }
            store_row_chunk(r, orow, col0, N, epilogue, dscale, fscale, out, out_dtype, ldo, vec_ok,
                            acc_out, ld_acc);
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
      } else {
        // partial tile -> slab sp (row-major M x N int32); summed by splitk_finalize
        int32_t* slab = slabs + int64_t(sp) * M * N;
#pragma unroll 1
        for (int c = grp; c < BN / 32; c += kGroups) {
          const int64_t col0 = int64_t(nb) * BN + c * 32;
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(tmem_base + ((quarter * 32) << 16) + uint32_t(acc * BN + c * 32), r);
          ptx::tmem_ld_wait();
          if (row < M && col0 < N) {
            int32_t* d = slab + row * N + col0;
            if (col0 + 32 <= N && (N & 3) == 0) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                __stcg(reinterpret_cast<int4*>(d + j),
                       make_int4(int(r[j]), int(r[j + 1]), int(r[j + 2]), int(r[j + 3])));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j < N) d[j] = int(r[j]);
            }
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  if (((warp >= 4 && warp < 8) || (!A4 && warp >= 8 && warp < 12)) && lane == 0)
    ptx::bulk_wait_read<0>();  // staging reads done before the CTA exits
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, Cfg::kTmemCols);
}

// CTA-pair variant (tcgen05 cta_group::2): a cluster of 2 CTAs on one TPC
// computes a 256 x BN tile.  CTA r stages A rows [128 r, 128 r + 128) and B
// rows [BN/2 r, BN/2 r + BN/2) of every K block in its own shared memory, and
// its TMEM holds its 128 accumulator rows; only the leader (rank 0) issues the
// MMAs.  Per SM that is 16 + BN/2*128/1024 KB of operands per 128-byte K block
// for 128 x BN MACs -- a third less L2->SM traffic than the 128 x BN single-CTA
// tile.  Pipelines: both producers wait on their own `empty` (the leader's MMA
// commit multicasts to both CTAs) and complete bytes on the LEADER's `full`;
// the MMA commit multicasts `tfull` to both CTAs; every epilogue warp of both
// CTAs arrives on the leader's `tempty`.
//
// Up to two independent products share one launch (the dX and dW GEMMs of a
// layer): units of problem 0 come first in the global unit numbering, and an
// optional host-built schedule (longest-processing-time first, per cluster)
// lists each cluster's units so long dW units and short dX units pack evenly.
struct PairProb {
  int M, N, K, groups, splits, tma_out, epilogue, out_dtype;
  int a4;  // A is packed int4 (map a[] boxes 64 bytes x 128 rows; converted in smem)
  const float* sa;
  const float* sb;
  double extra;
  void* out;
  int64_t ldo;
  int32_t* acc_out;
  int64_t ld_acc;
  int32_t* slabs;
  int unit0, units;
};
constexpr int kMaxSched = 11000;
struct alignas(64) PairParams {
  CUtensorMap a[2], b[2], o[2];
  PairProb p[2];
  int nprob, nsched;
  uint16_t off[129];
  uint16_t ids[kMaxSched];
};

template <int BN, int STAGES, bool A4ANY>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(A4ANY ? kThreadsA4 : kThreads, 1)
    gemm_i8_2sm_kernel(const __grid_constant__ PairParams P) {
  constexpr uint32_t kABytes = kBM * kBK;             // this CTA's 128 rows of A
  constexpr uint32_t kBBytes = (BN / 2) * kBK;        // this CTA's BN/2 rows of B
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;  // power of two >= 2*BN
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kABytes;
  uint8_t* stg = sB + STAGES * kBBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + kStgAll);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  // packed-A units: each CTA's packed A completes on its own `pfull`; its
  // converters then arrive on the LEADER's `aready` (4 warps x 2 CTAs).  These
  // two complete only on packed rounds, so every role tracks their phases per
  // stage (bit s of `pph`).
  uint64_t* pfull = tempty + 2;
  uint64_t* aready = pfull + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aready + STAGES);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_rank();
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    for (int q = 0; q < P.nprob; ++q) {
      ptx::tma_prefetch_desc(&P.a[q]);
      ptx::tma_prefetch_desc(&P.b[q]);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&pfull[s], 1);
      ptx::mbar_init(&aready[s], 2 * kConvWarps);  // converter warps x 2 CTAs
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, kTmemCols);
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barrier inits visible to the peer before any remote arrive / TMA
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent launch (see gemm_i8_kernel)

  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int total = P.p[0].units + (P.nprob > 1 ? P.p[1].units : 0);
  const int count = P.nsched ? int(P.off[cid + 1]) - int(P.off[cid]) : (total - cid + ncl - 1) / ncl;
  const uint32_t full_leader = ptx::mapa(ptx::smem_u32(full), 0);
  const uint32_t tempty_leader = ptx::mapa(ptx::smem_u32(tempty), 0);
  const uint32_t aready_leader = ptx::mapa(ptx::smem_u32(aready), 0);

  // unit i of this cluster -> (problem, tile, split, K-block range)
  struct U {
    int q, mb, nb, sp, kb0, kb1, nk_g;
  };
  auto unit = [&](int i) {
    const int u = P.nsched ? int(P.ids[P.off[cid] + i]) : cid + i * ncl;
    U r;
    r.q = (P.nprob > 1 && u >= P.p[1].unit0) ? 1 : 0;
    const PairProb& pr = P.p[r.q];
    const int local = u - pr.unit0;
    const int t = local / pr.splits;
    r.sp = local - t * pr.splits;
    const int num_n = (pr.N + BN - 1) / BN;
    r.mb = t / num_n;
    r.nb = t - r.mb * num_n;
    r.nk_g = (pr.K + kBK - 1) / kBK;
    const int nk = r.nk_g * pr.groups;
    r.kb0 = int(int64_t(r.sp) * nk / pr.splits);
    r.kb1 = int(int64_t(r.sp + 1) * nk / pr.splits);
    return r;
  };

  if (warp == 0) {
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < count; ++i) {
        const U w = unit(i);
        const CUtensorMap* ma = &P.a[w.q];
        const CUtensorMap* mb = &P.b[w.q];
        int g = w.kb0 / w.nk_g, kg = w.kb0 - g * w.nk_g;
        const bool a4 = A4ANY && P.p[w.q].a4;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          ptx::mbar_wait_sleep(&empty[stage], phase ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], a4 ? 2 * kBBytes : 2 * kStageBytes);
          const uint32_t fb = full_leader + uint32_t(stage) * 8u;
          if (a4) {
            // this CTA's packed A rows -> upper half of its A slot, completion on its own pfull
            ptx::mbar_arrive_expect_tx(&pfull[stage], kPackedA);
            ptx::tma_load_3d(sA + stage * kABytes + kPackedA, ma, &pfull[stage], kg * (kBK / 2),
                             w.mb * 2 * kBM + int(rank) * kBM, g);
          } else {
            ptx::tma_load_3d_2sm(sA + stage * kABytes, ma, fb, kg * kBK, w.mb * 2 * kBM + int(rank) * kBM, g);
          }
          ptx::tma_load_3d_2sm(sB + stage * kBBytes, mb, fb, kg * kBK, w.nb * BN + int(rank) * (BN / 2), g);
          if (++kg == w.nk_g) { kg = 0; ++g; }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_i8(2 * kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      uint32_t pph = 0;
      for (int i = 0; i < count; ++i) {
        const U w = unit(i);
        const bool a4 = A4ANY && P.p[w.q].a4;
        ptx::mbar_wait_sleep(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          if (a4) {
            ptx::mbar_wait(&aready[stage], (pph >> stage) & 1u);  // both CTAs' A converted
            pph ^= 1u << stage;
          }
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint64_t a_desc = ptx::desc_kmajor_sw128(ptx::smem_u32(sA + stage * kABytes));
            const uint64_t b_desc = ptx::desc_kmajor_sw128(ptx::smem_u32(sB + stage * kBBytes));
#pragma unroll
            for (int k = 0; k < kBK / 32; ++k)
              ptx::mma_i8_2sm(d_tmem, a_desc + uint64_t((k * 32) >> 4), b_desc + uint64_t((k * 32) >> 4), idesc,
                              (kb != w.kb0 || k != 0) ? 1u : 0u);
            ptx::mma_commit_2sm(&empty[stage], 0x3);
            if (kb == w.kb1 - 1) ptx::mma_commit_2sm(&tfull[acc], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (A4ANY && warp >= 8) {
    // converters (both CTAs): sign-extend this CTA's packed A rows in place
    const int ct = int(threadIdx.x) - 256;
    int stage = 0;
    uint32_t pph = 0;
    for (int i = 0; i < count; ++i) {
      const U w = unit(i);
      const bool a4 = P.p[w.q].a4 != 0;
      for (int kb = w.kb0; kb < w.kb1; ++kb) {
        if (a4) {
          ptx::mbar_wait(&pfull[stage], (pph >> stage) & 1u);
          pph ^= 1u << stage;
          convert_a4(sA + stage * kABytes, ct);
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_remote(aready_leader + uint32_t(stage) * 8u);
        }
        if (++stage == STAGES) stage = 0;
      }
    }
  } else if (warp >= 4 && warp < 8) {
    const uint32_t quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int i = 0; i < count; ++i) {
      const U w = unit(i);
      const PairProb& pr = P.p[w.q];
      const float comb = __fmul_rn(*pr.sa, *pr.sb);
      const double dscale = __dmul_rn(double(comb), pr.extra);
      const float fscale = float(dscale);
      const bool vec_ok = (pr.ldo % 8 == 0) && ((reinterpret_cast<uintptr_t>(pr.out) & 15) == 0);
      ptx::mbar_wait_sleep(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int64_t row = int64_t(w.mb) * 2 * kBM + int64_t(rank) * kBM + quarter * 32 + lane;
      const int32_t row0 = w.mb * 2 * kBM + int32_t(rank) * kBM + int32_t(quarter) * 32;
      uint8_t* wbuf = stg + quarter * kStgBytes;
      if (pr.splits == 1 && pr.tma_out && pr.out_dtype == kBF16) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; c += 2) {  // 32 x 64 tiles (128-byte rows)
          const int32_t col0 = w.nb * BN + c * 32;
          uint32_t r0[32], r1[32];
          ptx::tmem_ld_32x32b_x32(tmem_base + ((quarter * 32) << 16) + uint32_t(acc * BN + c * 32), r0);
          ptx::tmem_ld_32x32b_x32(tmem_base + ((quarter * 32) << 16) + uint32_t(acc * BN + c * 32 + 32), r1);
          ptx::tmem_ld_wait();
          if (lane == 0) ptx::bulk_wait_read<1>();
          __syncwarp();
          if (row0 < pr.M && col0 < pr.N)
            store_pair_tma_bf16(r0, r1, fscale, wbuf + ((c >> 1) & 1) * (kStgBytes / 2), lane, &P.o[w.q], col0,
                                row0);
        }
      } else
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        const int64_t col0 = int64_t(w.nb) * BN + c * 32;
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((quarter * 32) << 16) + uint32_t(acc * BN + c * 32), r);
        ptx::tmem_ld_wait();
        if (pr.splits == 1 && pr.tma_out) {
          if (lane == 0) ptx::bulk_wait_read<1>();
          __syncwarp();
          if (row0 < pr.M && col0 < pr.N)
            store_chunk_tma(r, fscale, pr.out_dtype, wbuf + (c & 1) * (kStgBytes / 2), lane, &P.o[w.q],
                            int32_t(col0), row0);
        } else if (row < pr.M && col0 < pr.N) {
          if (pr.splits == 1) {
            store_row_chunk(r, row, col0, pr.N, pr.epilogue, dscale, fscale, pr.out, pr.out_dtype, pr.ldo, vec_ok,
                            pr.acc_out, pr.ld_acc);
          } else {
            int32_t* d = pr.slabs + int64_t(w.sp) * pr.M * pr.N + row * pr.N + col0;
            if (col0 + 32 <= pr.N && (pr.N & 3) == 0) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                __stcg(reinterpret_cast<int4*>(d + j),
                       make_int4(int(r[j]), int(r[j + 1]), int(r[j + 2]), int(r[j + 3])));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j < pr.N) d[j] = int(r[j]);
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      // default-semantics remote arrive (as CUTLASS's 2-SM TMEM-empty arrive): the
      // release.cluster form compiled to a MEMBAR + ERRBAR per tile and warp
      if (lane == 0) ptx::mbar_arrive_remote(tempty_leader + uint32_t(acc) * 8u);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  if (warp >= 4 && warp < 8 && lane == 0) ptx::bulk_wait_read<0>();
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_2sm(tmem_base, kTmemCols);
}

// out[m, n] = dequant(sum_s slab[s][m, n]) (+ the exact int32 sum into acc_out).
// The slabs are summed in int64: a contraction longer than the int32-exact
// bound is planned as >= 2 splits each inside it (the reference accumulates in
// int64 up to MAX_K, quantize.py:21,167), and acc_out is then not requested.
__global__ void __launch_bounds__(256) splitk_finalize(const int32_t* __restrict__ slabs, int splits,
                                                       int M, int N, const float* __restrict__ sa,
                                                       const float* __restrict__ sb, double extra,
                                                       int epilogue, void* out, int out_dtype, int64_t ldo,
                                                       int32_t* acc_out, int64_t ld_acc, int vec) {
  const float comb = __fmul_rn(*sa, *sb);
  const double dscale = __dmul_rn(double(comb), extra);
  const float fscale = float(dscale);
  const int64_t plane = int64_t(M) * N;
  if (!vec) {
    // any N / output alignment (e.g. the 27 columns of an RGB stem's conv dW): one element per thread
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < plane; e += int64_t(gridDim.x) * blockDim.x) {
      long long a = __ldcs(slabs + e);
      for (int s = 1; s < splits; ++s) a += __ldcs(slabs + s * plane + e);
      const int64_t m = e / N, n = e - m * N;
      if (acc_out) acc_out[m * ld_acc + n] = int(a);
      if (!out) continue;
      const float v = epilogue == kEpiExact ? __double2float_rn(__dmul_rn(__ll2double_rn(a), dscale))
                                            : __fmul_rn(__ll2float_rn(a), fscale);
      if (out_dtype == kF32)
        static_cast<float*>(out)[m * ldo + n] = v;
      else
        static_cast<__nv_bfloat16*>(out)[m * ldo + n] = __float2bfloat16_rn(v);
    }
    return;
  }
  const int64_t nq = plane >> 2;  // vec: N % 4 == 0 and 16-byte aligned rows
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < nq; q += int64_t(gridDim.x) * blockDim.x) {
    const int4 t0 = __ldcs(reinterpret_cast<const int4*>(slabs) + q);
    long long a[4] = {t0.x, t0.y, t0.z, t0.w};
    for (int s = 1; s < splits; ++s) {
      const int4 v = __ldcs(reinterpret_cast<const int4*>(slabs + s * plane) + q);
      a[0] += v.x; a[1] += v.y; a[2] += v.z; a[3] += v.w;
    }
    const int64_t e = q << 2;
    const int64_t m = e / N, n = e - m * N;
    if (acc_out)
      *reinterpret_cast<int4*>(acc_out + m * ld_acc + n) = make_int4(int(a[0]), int(a[1]), int(a[2]), int(a[3]));
    if (!out) continue;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      v[j] = epilogue == kEpiExact ? __double2float_rn(__dmul_rn(__ll2double_rn(a[j]), dscale))
                                   : __fmul_rn(__ll2float_rn(a[j]), fscale);
    if (out_dtype == kF32) {
      *reinterpret_cast<float4*>(static_cast<float*>(out) + m * ldo + n) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]), p1 = __floats2bfloat162_rn(v[2], v[3]);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t*>(&p0);
      w.y = *reinterpret_cast<uint32_t*>(&p1);
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(out) + m * ldo + n) = w;
    }
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 3-D map (K, rows, groups): OOB rows / K columns of a group are zero-filled,
// so ragged tiles never read a neighbouring group's data.
bool make_map(CUtensorMap* map, const int8_t* ptr, int64_t rows, int64_t k, int64_t ld,
              int64_t groups, int64_t gstride, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {cuuint64_t(k), cuuint64_t(rows), cuuint64_t(groups)};
  cuuint64_t strides[2] = {cuuint64_t(ld), cuuint64_t(groups > 1 ? gstride : ld * rows)};
  cuuint32_t box[3] = {uint32_t(kBK), box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Packed int4 A: (ceil(K/2) bytes, rows, groups), 64-byte x 128-row boxes (one
// stage of K = 128 codes), no swizzle -- the converter warps write the SW128 tile.
bool make_map_a4(CUtensorMap* map, const int8_t* ptr, int64_t rows, int64_t k, int64_t ld, int64_t groups,
                 int64_t gstride) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {cuuint64_t((k + 1) / 2), cuuint64_t(rows), cuuint64_t(groups)};
  cuuint64_t strides[2] = {cuuint64_t(ld), cuuint64_t(groups > 1 ? gstride : ld * rows)};
  cuuint32_t box[3] = {uint32_t(kBK / 2), uint32_t(kBM), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Store map of the output for the TMA epilogue: (N, M) with row stride ldo,
// 32-row boxes of 128-byte rows (32 fp32 / 64 bf16 columns), SW128 as
// store_chunk_tma / store_pair_tma_bf16 write them.  False = use the direct
// store epilogue (exact fp64 dequant, int32 accumulator dump, split-K slabs or
// an output TMA cannot describe).
bool make_out_map(CUtensorMap* map, void* out, int out_dtype, int64_t M, int64_t N, int64_t ldo, int epilogue,
                  const int32_t* acc_out, int splits) {
  if (!out || acc_out || splits != 1 || epilogue != kEpiFast) return false;
  static const int knob_direct = env_knob("HLQ_GEMM_DIRECT_OUT");  // development A/B
  if (knob_direct == 1) return false;
  const int64_t esz = out_dtype == kBF16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(out) % 16) || (ldo * esz) % 16 || M <= 0 || N <= 0) return false;
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(M)};
  cuuint64_t strides[1] = {cuuint64_t(ldo * esz)};
  cuuint32_t box[2] = {out_dtype == kBF16 ? 64u : 32u, 32};  // 128-byte rows either way
  cuuint32_t es[2] = {1, 1};
  return fn(map, out_dtype == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out,
            dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool encode_tensor_map(void* map, int dtype, int rank, const void* ptr, const uint64_t* dims,
                       const uint64_t* strides_bytes, const uint32_t* box, int swizzle_128b) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || rank < 1 || rank > 5) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i < rank - 1) s[i] = strides_bytes[i];
  }
  const CUtensorMapDataType t = dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                : dtype == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                             : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  return fn(static_cast<CUtensorMap*>(map), t, cuuint32_t(rank), const_cast<void*>(ptr), d, s, b, e,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            swizzle_128b ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

// Programmatic dependent launch (HLQ_PDL=0 disables): the GEMM's CTAs may start
// their prologue (barriers, TMEM, descriptor prefetch) while the previous
// kernel on the stream drains, and griddepcontrol.wait before touching its
// outputs; the fused transforms trigger their dependents as each CTA finishes.
void pdl_attr(cudaLaunchAttribute& a) {
  static const int off = env_knob("HLQ_PDL");
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = off == 0 ? 0 : 1;
}

template <int BN, int STAGES, bool A4 = false>
int run_maps(const CUtensorMap& ma, const CUtensorMap& mb, int64_t M, int64_t N, int64_t K, int64_t groups,
             const float* sa, const float* sb, double extra, int epilogue, void* out, int out_dtype,
             int64_t ldo, int32_t* acc_out, int64_t ld_acc, int splits, void* ws, const ConvGeo& geo,
             cudaStream_t stream) {
  using Cfg = GemmCfg<BN, STAGES>;
  static std::atomic<unsigned long long> attr_set{0};  // per template instance and device
  {
    cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(gemm_i8_kernel<BN, STAGES, A4>), int(Cfg::kSmem),
                                   attr_set);
    if (e != cudaSuccess) return int(e);
  }
  const int64_t tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  int32_t* slabs = splits > 1 ? static_cast<int32_t*>(ws) : nullptr;
  const int64_t units = tiles * splits;
  const int grid = int(units < num_sms() ? units : num_sms());
  CUtensorMap mo;
  // strided conv phases scatter their rows: the direct-store epilogue
  const int tma_out =
      (geo.conv && geo.s > 1) ? 0 : (make_out_map(&mo, out, out_dtype, M, N, ldo, epilogue, acc_out, splits) ? 1 : 0);
  if (!tma_out) mo = ma;  // unused
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(A4 ? kThreadsA4 : kThreadsE2);
    cfg.dynamicSmemBytes = Cfg::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    pdl_attr(at[0]);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, gemm_i8_kernel<BN, STAGES, A4>, ma, mb, mo, tma_out, int(M), int(N), int(K),
                       int(groups), sa, sb, extra, epilogue, out, out_dtype, ldo, acc_out, ld_acc, splits, slabs,
                       geo);
  }
  if (splits > 1) {
    const int64_t nq = M * N / 4;
    int fgrid = int((nq + 255) / 256);
    if (fgrid > num_sms() * 8) fgrid = num_sms() * 8;
    const int vec = (N % 4 == 0) && (ldo % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                    (ld_acc % 4 == 0) && (reinterpret_cast<uintptr_t>(acc_out) % 16 == 0);
    splitk_finalize<<<fgrid, 256, 0, stream>>>(slabs, splits, int(M), int(N), sa, sb, extra, epilogue, out,
                                               out_dtype, ldo, acc_out, ld_acc, vec);
  }
  return int(cudaGetLastError());
}

template <int BN, int STAGES>
int run(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
        int64_t groups, int64_t a_gstride, int64_t b_gstride, const float* sa, const float* sb, double extra, int epilogue, void* out, int out_dtype,
        int64_t ldo, int32_t* acc_out, int64_t ld_acc, int splits, void* ws, cudaStream_t stream, bool a4) {
  CUtensorMap ma, mb;
  const bool okA = a4 ? make_map_a4(&ma, A, M, K, lda, groups, a_gstride)
                      : make_map(&ma, A, M, K, lda, groups, a_gstride, kBM);
  if (!okA || !make_map(&mb, B, N, K, ldb, groups, b_gstride, BN)) return -1;
  const ConvGeo geo{0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0};
  if (a4)  // the widened A holds 16 * code: 1/16 in the dequant scale (exact)
    return run_maps<BN, STAGES, true>(ma, mb, M, N, K, groups, sa, sb, extra * 0.0625, epilogue, out, out_dtype,
                                      ldo, acc_out, ld_acc, splits, ws, geo, stream);
  return run_maps<BN, STAGES>(ma, mb, M, N, K, groups, sa, sb, extra, epilogue, out, out_dtype, ldo, acc_out,
                              ld_acc, splits, ws, geo, stream);
}

struct PairSpec {  // one product for the CTA-pair kernel
  const int8_t* A;
  int64_t lda;
  const int8_t* B;
  int64_t ldb;
  int64_t M, N, K, groups, a_gstride, b_gstride;
  const float* sa;
  const float* sb;
  double extra;
  int epilogue;
  void* out;
  int out_dtype;
  int64_t ldo;
  int32_t* acc_out;
  int64_t ld_acc;
  int splits;
  void* ws;
  int a4;  // A packed int4
};

template <int BN>
bool fill_prob(PairParams& P, int q, const PairSpec& s, int unit0) {
  const bool okA = s.a4 ? make_map_a4(&P.a[q], s.A, s.M, s.K, s.lda, s.groups, s.a_gstride)
                        : make_map(&P.a[q], s.A, s.M, s.K, s.lda, s.groups, s.a_gstride, kBM);
  if (!okA || !make_map(&P.b[q], s.B, s.N, s.K, s.ldb, s.groups, s.b_gstride, BN / 2)) return false;
  PairProb& p = P.p[q];
  p.a4 = s.a4;
  p.M = int(s.M); p.N = int(s.N); p.K = int(s.K); p.groups = int(s.groups); p.splits = s.splits;
  p.tma_out = make_out_map(&P.o[q], s.out, s.out_dtype, s.M, s.N, s.ldo, s.epilogue, s.acc_out, s.splits) ? 1 : 0;
  if (!p.tma_out) P.o[q] = P.a[q];  // unused
  p.epilogue = s.epilogue; p.out_dtype = s.out_dtype; p.sa = s.sa; p.sb = s.sb;
  p.extra = s.a4 ? s.extra * 0.0625 : s.extra;  // packed A is widened to 16 * code
  p.out = s.out; p.ldo = s.ldo; p.acc_out = s.acc_out; p.ld_acc = s.ld_acc;
  p.slabs = s.splits > 1 ? static_cast<int32_t*>(s.ws) : nullptr;
  p.unit0 = unit0;
  p.units = int(((s.M + 2 * kBM - 1) / (2 * kBM)) * ((s.N + BN - 1) / BN) * s.splits);
  return true;
}

// Longest-processing-time-first static schedule over the clusters (cost of a
// unit = its K blocks + a fixed epilogue / pipeline-fill term).  false if the
// table does not fit the kernel parameters (then: round-robin).
bool lpt_schedule(PairParams& P, int ncl) {
  const int total = P.p[0].units + (P.nprob > 1 ? P.p[1].units : 0);
  if (total > kMaxSched || ncl > 128 || total > 65535) return false;
  std::vector<std::pair<int, int>> cost(total);  // (cost, unit)
  for (int u = 0; u < total; ++u) {
    const PairProb& pr = P.p[(P.nprob > 1 && u >= P.p[1].unit0) ? 1 : 0];
    const int nk = ((pr.K + kBK - 1) / kBK) * pr.groups / pr.splits;
    // fixed per-unit term (epilogue, pipeline fill): 2 measured best for the fc2
    // dW + dX mix (74 us vs 78 us at 4 and 0; fc1 / qkv unchanged)
    static const int knob_epi = env_knob("HLQ_GEMM_LPT_EPI");  // development sweeps
    cost[u] = {nk + (knob_epi >= 0 ? knob_epi : 2), u};
  }
  std::stable_sort(cost.begin(), cost.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  std::vector<int64_t> load(ncl, 0);
  std::vector<std::vector<uint16_t>> lists(ncl);
  for (const auto& cu : cost) {
    int best = 0;
    for (int c = 1; c < ncl; ++c)
      if (load[c] < load[best]) best = c;
    load[best] += cu.first;
    lists[best].push_back(uint16_t(cu.second));
  }
  int o = 0;
  for (int c = 0; c < ncl; ++c) {
    P.off[c] = uint16_t(o);
    for (uint16_t u : lists[c]) P.ids[o++] = u;
  }
  P.off[ncl] = uint16_t(o);
  P.nsched = 1;
  return true;
}

template <int BN, int STAGES>
int run_2sm_specs(const PairSpec* specs, int n, cudaStream_t stream) {
  constexpr size_t kSmem = size_t(STAGES) * (kBM * kBK + (BN / 2) * kBK) + kStgAll + 1024 + 512;
  static PairParams P;  // host staging (large); launches copy it into the parameter buffer
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  memset(&P, 0, sizeof(P));
  P.nprob = n;
  int unit0 = 0;
  for (int q = 0; q < n; ++q) {
    if (!fill_prob<BN>(P, q, specs[q], unit0)) return -1;
    unit0 += P.p[q].units;
  }
  bool any_a4 = false;
  for (int q = 0; q < n; ++q) any_a4 = any_a4 || specs[q].a4;
  static std::atomic<unsigned long long> attr_set{0}, attr_set4{0};  // per template instance and device
  {
    cudaError_t e = any_a4 ? smem_attr_once(reinterpret_cast<const void*>(gemm_i8_2sm_kernel<BN, STAGES, true>),
                                            int(kSmem), attr_set4)
                           : smem_attr_once(reinterpret_cast<const void*>(gemm_i8_2sm_kernel<BN, STAGES, false>),
                                            int(kSmem), attr_set);
    if (e != cudaSuccess) return int(e);
  }
  const int64_t pairs = num_sms() / 2;
  const int ncl = int(unit0 < pairs ? unit0 : pairs);
  if (n > 1) lpt_schedule(P, ncl);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * ncl);
    cfg.blockDim = dim3(any_a4 ? kThreadsA4 : kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    pdl_attr(at[0]);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (any_a4)
      cudaLaunchKernelEx(&cfg, gemm_i8_2sm_kernel<BN, STAGES, true>, P);
    else
      cudaLaunchKernelEx(&cfg, gemm_i8_2sm_kernel<BN, STAGES, false>, P);
  }
  for (int q = 0; q < n; ++q) {
    const PairSpec& s = specs[q];
    if (s.splits > 1) {
      const int64_t nq = s.M * s.N / 4;
      int fgrid = int((nq + 255) / 256);
      if (fgrid > num_sms() * 8) fgrid = num_sms() * 8;
      const int vec = (s.N % 4 == 0) && (s.ldo % 4 == 0) && (reinterpret_cast<uintptr_t>(s.out) % 16 == 0) &&
                      (s.ld_acc % 4 == 0) && (reinterpret_cast<uintptr_t>(s.acc_out) % 16 == 0);
      splitk_finalize<<<fgrid, 256, 0, stream>>>(static_cast<int32_t*>(s.ws), s.splits, int(s.M), int(s.N), s.sa,
                                                 s.sb, s.a4 ? s.extra * 0.0625 : s.extra, s.epilogue, s.out,
                                                 s.out_dtype, s.ldo, s.acc_out, s.ld_acc, vec);
    }
  }
  return int(cudaGetLastError());
}

template <int BN, int STAGES>
int run_2sm(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
            int64_t groups, int64_t a_gstride, int64_t b_gstride, const float* sa, const float* sb, double extra,
            int epilogue, void* out, int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc, int splits,
            void* ws, cudaStream_t stream, bool a4) {
  const PairSpec s{A, lda, B, ldb, M, N, K, groups, a_gstride, b_gstride, sa, sb, extra, epilogue, out, out_dtype,
                   ldo, acc_out, ld_acc, splits, ws, a4 ? 1 : 0};
  return run_2sm_specs<BN, STAGES>(&s, 1, stream);
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
}

// Tile width, split count and workspace bytes for one GEMM.  Split-K only when
// the output has too few tiles to fill the SMs and K is long (the dW products:
// M = O, N = I, K = projected tokens).
struct GemmPlan {
  int bn, splits;
  size_t ws;
  bool pair;  // CTA-pair (cta_group::2) 256 x bn tiles
};

GemmPlan finish_plan(GemmPlan p, int64_t M, int64_t N, bool allow_split);
GemmPlan plan_gemm_base(int64_t M, int64_t N, int64_t K, int64_t groups, bool allow_split);

// min_splits > 1: the contraction exceeds the int32-exact bound, so it must run
// as at least that many K chunks (int32 partial slabs, int64 finalize).
GemmPlan plan_gemm(int64_t M, int64_t N, int64_t K, int64_t groups, bool allow_split, int min_splits = 1) {
  GemmPlan p = plan_gemm_base(M, N, K, groups, allow_split || min_splits > 1);
  if (min_splits > p.splits) {
    p.splits = min_splits;
    p.ws = size_t(p.splits) * M * N * 4;
  }
  return p;
}

GemmPlan plan_gemm_base(int64_t M, int64_t N, int64_t K, int64_t groups, bool allow_split) {
  const int64_t m_tiles = (M + kBM - 1) / kBM;
  const int64_t wide_tiles = m_tiles * ((N + 255) / 256);
  const int64_t nk = ((K + kBK - 1) / kBK) * groups;
  const int64_t sms = num_sms();
  GemmPlan p{128, 1, 0, false};
  if (N > 128 && wide_tiles >= sms) p.bn = 256;
  const int64_t tiles = m_tiles * ((N + p.bn - 1) / p.bn);
  // Long contractions with enough rows run as CTA pairs (cta_group::2, 256-row
  // tiles: a third less operand traffic per MAC).  Tile width by a makespan
  // model: rounds of pair units x relative unit cost (a 256 x 128 unit costs
  // ~0.6 of a 256 x 256 one; tools/gemm_sweep.py, B200).  Wide outputs (N >=
  // 2048) take pairs at any K: a single CTA's 128 x 256 tile moves ~117 KB of
  // shared memory per 128-byte K block (TMA in, MMA operand reads, epilogue
  // staging) against ~545 cycles of MMA -- shared-memory bound at ~55 % tensor
  // (ncu, fc2 dX); the pair halves the B traffic per SM (fc2 dX 63.5 -> 55 us).
  const int64_t tiles128 = m_tiles * ((N + 127) / 128);
  const bool split_case = allow_split && 2 * tiles128 <= sms && nk >= 16;
  if (!split_case && (nk >= 16 || (N >= 2048 && nk >= 2)) && M >= 2 * kBM && sms >= 2) {
    const int64_t pairs = sms / 2, pm = (M + 2 * kBM - 1) / (2 * kBM);
    const int64_t u256 = pm * ((N + 255) / 256), u192 = pm * ((N + 191) / 192), u128 = pm * ((N + 127) / 128);
    const double t256 = double((u256 + pairs - 1) / pairs), t192 = 0.9 * double((u192 + pairs - 1) / pairs),
                 t128 = 0.6 * double((u128 + pairs - 1) / pairs);
    p.pair = true;
    p.bn = 128;
    double best = t128;
    if (N > 128 && t192 < best) { best = t192; p.bn = 192; }
    if (N > 128 && t256 <= best) p.bn = 256;
    return finish_plan(p, M, N, allow_split);
  }
  // Split-K only for products that fill less than half the SMs (e.g. the ViT
  // proj dW, 36 tiles of K = 13312): the slab round trip costs ~6 us per split
  // at fc1 size, which outweighs the wave gain once >= half the SMs are busy
  // (tools/gemm_sweep.py, B200).  (the finalize pass reads 16-byte int32 quads:
  // N % 4 == 0)
  if (allow_split && 2 * tiles <= sms && nk >= 16) {
    int64_t sp = sms / tiles;
    // the cap is the int32 slab round trip (splits x M x N x 4 bytes written and
    // re-read): 4 splits at ViT dW sizes (9.4 MB per slab), up to 64 for the
    // small-output, very long-K products of conv wgrad (ResNet CIFAR stem dW:
    // 64 x 27 outputs, K = 131072 -- one tile, 4 splits left 144 SMs idle)
    int64_t cap = (int64_t(64) << 20) / (M * N * 4);
    cap = cap < 4 ? 4 : (cap > 64 ? 64 : cap);
    if (sp > cap) sp = cap;
    while (sp > 1 && nk / sp < 8) --sp;
    p.splits = int(sp);
  }
  return finish_plan(p, M, N, allow_split);
}

// tuning knobs (development sweeps): HLQ_GEMM_SPLITS=s forces s splits (1 = off),
// HLQ_GEMM_BN=128|256 forces the tile width, HLQ_GEMM_PAIR=0|1 the CTA-pair kernel
GemmPlan finish_plan(GemmPlan p, int64_t M, int64_t N, bool allow_split) {
  static const int knob_bn = env_knob("HLQ_GEMM_BN"), knob_splits = env_knob("HLQ_GEMM_SPLITS"),
                   knob_pair = env_knob("HLQ_GEMM_PAIR");
  if (knob_bn == 128 || ((knob_bn == 256 || knob_bn == 192) && N > 128)) p.bn = knob_bn;
  if (knob_splits >= 1 && knob_splits <= 64 && allow_split) p.splits = knob_splits;
  if (knob_pair >= 0) p.pair = knob_pair != 0;
  if (p.splits > 1) p.ws = size_t(p.splits) * M * N * 4;
  return p;
}

}  // namespace

int launch_gemm_i8_pair2(const GemmDesc* d, cudaStream_t stream) {
  // both products as CTA-pair units of one launch (LPT-scheduled); the caller
  // checked that both have long contractions (>= 16 K blocks) and >= 256 rows
  const int bn = (d[0].N > 128 && d[1].N > 128) ? 256 : 128;
  PairSpec s[2];
  for (int q = 0; q < 2; ++q)
    s[q] = PairSpec{d[q].A, d[q].lda, d[q].B, d[q].ldb, d[q].M, d[q].N, d[q].K, d[q].groups, d[q].a_gstride,
                    d[q].b_gstride, d[q].sa, d[q].sb, d[q].extra, d[q].epilogue, d[q].out, d[q].out_dtype,
                    d[q].ldo, d[q].acc_out, d[q].ld_acc, 1, nullptr, d[q].a4};
  if (bn == 256) return run_2sm_specs<256, 6>(s, 2, stream);
  return run_2sm_specs<128, 8>(s, 2, stream);
}

bool gemm_i8_pair2_eligible(const GemmDesc* d) {
  static const int min_nk = env_knob("HLQ_GEMM_PAIR_MINK") >= 0 ? env_knob("HLQ_GEMM_PAIR_MINK") : 16;  // sweeps
  static const int knob_fuse2 = env_knob("HLQ_GEMM_FUSE2");
  // both products run as 256-row pair units; a short contraction qualifies when
  // its output is wide (N >= 2048: the pair's halved B traffic pays at any K,
  // plan_gemm_base) -- the ViT fc2 dX (K = 768, N = 3072) with its dW: 78 us
  // fused vs 91 us as two launches
  for (int q = 0; q < 2; ++q) {
    const int64_t nk = ((d[q].K + kBK - 1) / kBK) * d[q].groups;
    if ((nk < min_nk && !(d[q].N >= 2048 && nk >= 2)) || d[q].M < 2 * kBM) return false;
  }
  if (knob_fuse2 >= 0) return knob_fuse2 != 0;
  return true;
}

size_t gemm_i8_ws_bytes(int64_t M, int64_t N, int64_t K, int64_t groups, int min_splits) {
  return plan_gemm(M, N, K, groups, true, min_splits).ws;
}

int launch_gemm_i8(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int64_t M, int64_t N,
                   int64_t K, int64_t groups, int64_t a_gstride, int64_t b_gstride,
                   const float* sa, const float* sb, double extra, int epilogue,
                   void* out, int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc,
                   void* ws, size_t ws_bytes, cudaStream_t stream, int min_splits, bool a4) {
  GemmPlan p = plan_gemm(M, N, K, groups, true, min_splits);
  const bool vec_out = (ldo % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                       (ld_acc % 4 == 0) && (reinterpret_cast<uintptr_t>(acc_out) % 16 == 0);
  (void)vec_out;  // splitk_finalize has a scalar path for any N / output alignment
  if (p.splits > 1 && (ws == nullptr || ws_bytes < p.ws || (reinterpret_cast<uintptr_t>(ws) % 16))) {
    if (min_splits > 1) return -2;  // a long contraction cannot run without its chunk slabs
    p = plan_gemm(M, N, K, groups, false);
  }
  if (p.pair) {
    if (p.bn == 256)
      return run_2sm<256, 6>(A, lda, B, ldb, M, N, K, groups, a_gstride, b_gstride, sa, sb, extra, epilogue, out,
                             out_dtype, ldo, acc_out, ld_acc, p.splits, ws, stream, a4);
    if (p.bn == 192)
      return run_2sm<192, 6>(A, lda, B, ldb, M, N, K, groups, a_gstride, b_gstride, sa, sb, extra, epilogue, out,
                             out_dtype, ldo, acc_out, ld_acc, p.splits, ws, stream, a4);
    return run_2sm<128, 8>(A, lda, B, ldb, M, N, K, groups, a_gstride, b_gstride, sa, sb, extra, epilogue, out,
                           out_dtype, ldo, acc_out, ld_acc, p.splits, ws, stream, a4);
  }
  if (p.bn == 256)
    return run<256, 4>(A, lda, B, ldb, M, N, K, groups, a_gstride, b_gstride, sa, sb, extra, epilogue, out,
                       out_dtype, ldo, acc_out, ld_acc, p.splits, ws, stream, a4);
  return run<128, 6>(A, lda, B, ldb, M, N, K, groups, a_gstride, b_gstride, sa, sb, extra, epilogue, out,
                     out_dtype, ldo, acc_out, ld_acc, p.splits, ws, stream, a4);
}

int launch_conv_dgrad_i8(const int8_t* G, int64_t ldg, int64_t B, int64_t Ho, int64_t Wo, int64_t O,
                         const int8_t* Wc, int64_t ldw, int64_t C, int k, int stride, int pad, int64_t H,
                         int64_t W, const float* sa, const float* sb, int epilogue, void* out, int out_dtype,
                         int64_t ldo, int32_t* acc_out, int64_t ld_acc, cudaStream_t stream) {
  EncodeIm2colFn enc = encode_im2col_fn();
  EncodeTiledFn tenc = encode_fn();
  if (!enc || !tenc) return -1;
  const int s = stride;
  O = (O + 15) & ~int64_t(15);  // the contraction runs over the padded HT blocks (codes of pad16(O))
  const int nkc = int((O + kBK - 1) / kBK);
  // phases with output pixels but no tap get no contribution: zero dX (and the acc dump) first
  bool empty_phase = false;
  for (int ph = 0; ph < s; ++ph)
    for (int pw = 0; pw < s; ++pw) {
      const int i0 = (ph + pad) % s, j0 = (pw + pad) % s;
      if ((i0 >= k || j0 >= k) && ph < H && pw < W) empty_phase = true;
    }
  if (empty_phase) {
    const size_t esz = out_dtype == kBF16 ? 2 : 4;
    if (out && cudaMemsetAsync(out, 0, size_t(B * H * W) * ldo * esz, stream) != cudaSuccess) return -1;
    if (acc_out && cudaMemsetAsync(acc_out, 0, size_t(B * H * W) * ld_acc * 4, stream) != cudaSuccess) return -1;
  }
  for (int ph = 0; ph < s; ++ph)
    for (int pw = 0; pw < s; ++pw) {
      const int i0 = (ph + pad) % s, j0 = (pw + pad) % s;
      const int64_t Hp = (H - ph + s - 1) / s, Wp = (W - pw + s - 1) / s;
      if (i0 >= k || j0 >= k || Hp <= 0 || Wp <= 0) continue;
      const int kh = (k - i0 + s - 1) / s, kw = (k - j0 + s - 1) / s;
      const int dh = (ph + pad - i0) / s, dw = (pw + pad - j0) / s;
      const int lo_h = dh - kh + 1, lo_w = dw - kw + 1;
      CUtensorMap ma, mb;
      {
        // gy codes as NHWC int8: dims (O, Wo, Ho, B), pixel stride ldg bytes; the traversal
        // walks the Hp x Wp phase grid: upper corner = lower + (phase extent - gy extent)
        cuuint64_t dims[4] = {cuuint64_t(O), cuuint64_t(Wo), cuuint64_t(Ho), cuuint64_t(B)};
        cuuint64_t strides[3] = {cuuint64_t(ldg), cuuint64_t(ldg * Wo), cuuint64_t(ldg * Wo * Ho)};
        const int lower[2] = {lo_w, lo_h};
        const int upper[2] = {int(lo_w + Wp - Wo), int(lo_h + Hp - Ho)};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(G), dims, strides, lower, upper,
                cuuint32_t(kBK), cuuint32_t(kBM), es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return -1;
      }
      const int64_t M = B * Hp * Wp;
      // narrow outputs (C <= 64, the ResNet CIFAR stage 1): 128 x 64 tiles, no half-empty N
      static const int knob_bn64 = env_knob("HLQ_GEMM_DGRAD_BN64");  // development A/B
      const int bn = (C > 128 && ((M + kBM - 1) / kBM) * ((C + 255) / 256) >= num_sms()) ? 256
                     : (C <= 64 && knob_bn64 != 0) ? 64 : 128;
      {
        // W codes (C*k*k rows of ldw bytes, K = o), this phase's taps (i0 + s ti, j0 + s tj):
        // dims (O, kw, kh, C), strides (s ldw, s k ldw, k^2 ldw)
        cuuint64_t dims[4] = {cuuint64_t(O), cuuint64_t(kw), cuuint64_t(kh), cuuint64_t(C)};
        cuuint64_t strides[3] = {cuuint64_t(ldw * s), cuuint64_t(ldw * s * k), cuuint64_t(ldw * k * k)};
        cuuint32_t box[4] = {cuuint32_t(kBK), 1, 1, cuuint32_t(bn)};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (tenc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(Wc + (int64_t(i0) * k + j0) * ldw), dims,
                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return -1;
      }
      const ConvGeo geo{1, int(Hp), int(Wp), kh, kw, lo_h, lo_w, nkc, s, ph, pw, int(H), int(W)};
      const int e = bn == 256 ? run_maps<256, 4>(ma, mb, M, C, O, 1, sa, sb, 1.0, epilogue, out, out_dtype, ldo,
                                                 acc_out, ld_acc, 1, nullptr, geo, stream)
                    : bn == 64  ? run_maps<64, 8>(ma, mb, M, C, O, 1, sa, sb, 1.0, epilogue, out, out_dtype, ldo,
                                                  acc_out, ld_acc, 1, nullptr, geo, stream)
                                : run_maps<128, 6>(ma, mb, M, C, O, 1, sa, sb, 1.0, epilogue, out, out_dtype, ldo,
                                                   acc_out, ld_acc, 1, nullptr, geo, stream);
      if (e != 0) return e;
    }
  return 0;
}

}  // namespace hlq
