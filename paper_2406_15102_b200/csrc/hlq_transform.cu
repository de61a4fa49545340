// Block-Hadamard transform + per-tensor amax + pseudo-stochastic quantizer
// (TMA-fed, the production path; hlq_transform_fallback.cu handles sources a
// tensor map cannot describe).
//
// Operands of the HLQ backward, all produced here:
//   gx left   Q4(HT_O(gy))   HT along the contiguous axis, codes (T, pad16(O))  backprop.py:362,367
//   gx right  Q4(HT_O(W))    HT along rows of W, codes written (I, pad16(O))    backprop.py:363,368
//   gw left   Q8(P gy)^T     rank-r projection along tokens, codes (O, K)       backprop.py:401-407
//   gw right  Q8(P X)        ACBP, rank-r projection along tokens, (I, K)       backprop.py:373-385
// Everything the tensor-core GEMM consumes is written K-major.
//
// Source view: S segments x R rows x C cols (row stride ld, segment stride).
// A "step" is one 16-row projection block x 256 columns.  Per CTA:
//   warp 4      TMA producer: one cp.async.bulk.tensor.3d per step into a
//               4-stage shared-memory ring (out-of-range rows / columns of the
//               box are zero-filled by the TMA unit = the reference's padding);
//   warps 0..3  consumers, per step:
//               phase 1: 256 (row, 16-col block) pieces, 2 per thread: the
//                        column-direction FWHT -> gx statistics / codes;
//               phase 2: 128 column pairs, 1 per thread: the row-direction
//                        FWHT (f32x2 lanes = the two columns, dead butterflies
//                        pruned for compile-time basis sets) -> gw statistics /
//                        codes staged in smem and flushed per work item as
//                        >= 32-byte runs of the K-major output rows.
// gy is therefore read once per pass for BOTH products ("dual" mode).
//
// Two passes: STATS (max|w| and min nonzero |w| of the transformed values,
// max-reduced on their IEEE bits) then QUANT.
//
// Bit-exactness (hadamard.py:121-134, quantize.py:94-145):
//  * butterfly stages h = 1, 2, 4, 8, (lower, upper) = (a + b, a - b), fp32 RN
//    (pairing two independent lanes in one f32x2 op changes nothing per lane);
//  * the reference multiplies by 0.25 then divides by s.  We keep w = 4v and
//    divide by d = s/512: Q = RN(w/d) = 2048 * RN(v/s) exactly (power-of-two
//    rescalings are exact for normal numbers), with the reciprocal-FMA division
//    Q = fma(fma(-Q0, d, w), r, Q0), r = RN(1/d), Q0 = RN(w r) -- verified
//    equal to IEEE division on 2.8e9 pairs inside the guard |w| >= 2^-100,
//    |Q| >= 2^-100, 2^-125 < d < 2^125 (tools/verify_fast_div.c).  The STATS
//    pass records min nonzero |w| so the QUANT pass checks the guard once per
//    tensor and otherwise falls back to the literal IEEE-division formula;
//  * code = lo + [frac*2048 > u] = ceil((Q - u) / 2048), evaluated as
//    RU(RU(Q - u) * 2^-11 + 1.5*2^23): the low bits of that float's pattern
//    are the two's-complement code -- no conversion instructions; the clip to
//    +-qmax runs on packed s16 lanes;
//  * the draw u = bits(v) & 0x7FF equals bits(w) & 0x7FF (same mantissa).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "hlq_internal.h"
#include "hlq_ptx.cuh"
#include "hlq_quant.cuh"

namespace hlq {

namespace {

using namespace dev;

constexpr int kCols = 256;       // columns per step
constexpr int kConsumers = 128;  // 4 consumer warps
constexpr int kThreads = kConsumers + 32;
constexpr int kStages = 4;

template <typename T>
struct Tr;
template <>
struct Tr<float> {
  static constexpr int kRow = kCols * 4;
  static constexpr int kDtype = 2;
};
template <>
struct Tr<__nv_bfloat16> {
  static constexpr int kRow = kCols * 2;
  static constexpr int kDtype = 1;
};

struct Args {
  int rows, cols, nblk, total_blocks, nb, ncol_tiles, items, rank;
  uint32_t bitmap;
  int bits_gx, bits_gw;
  uint32_t* stats;  // [0,1] gx, [2,3] gw
  int8_t* dst_gx;
  int64_t ld_gx;
  int8_t* dst_gw;
  int64_t ld_gw;
  float* scale_gx;
  float* scale_gw;
  int cstride;  // bytes per column in the code staging buffer
};

// (item, block) steps of this CTA with 32-bit counters; divisions once per item.
struct StepIter {
  int item, bl, nbl, gb0, col0, s, blk;
  __device__ __forceinline__ void start(const Args& a) {
    if (item >= a.items) return;
    const int g = item / a.ncol_tiles;
    col0 = (item - g * a.ncol_tiles) * kCols;
    gb0 = g * a.nb;
    nbl = min(a.nb, a.total_blocks - gb0);
    bl = 0;
    s = gb0 / a.nblk;
    blk = gb0 - s * a.nblk;
  }
  __device__ __forceinline__ void next(const Args& a) {
    if (++bl == nbl) {
      item += gridDim.x;
      start(a);
    } else if (++blk == a.nblk) {
      blk = 0;
      ++s;
    }
  }
};

// 16 elements of one row piece from the staged tile -> fp32
template <typename T>
__device__ __forceinline__ void read16(uint32_t p, float (&v)[16]) {
  if (sizeof(T) == 2) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint4 t = ptx::lds128(p + 16 * q);
      const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) { v[8 * q + 2 * k] = bf_lo(w[k]); v[8 * q + 2 * k + 1] = bf_hi(w[k]); }
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 t = ptx::lds128(p + 16 * q);
      v[4 * q] = __uint_as_float(t.x); v[4 * q + 1] = __uint_as_float(t.y);
      v[4 * q + 2] = __uint_as_float(t.z); v[4 * q + 3] = __uint_as_float(t.w);
    }
  }
}

template <typename T, int MODE, bool GX, bool GW, int BM, bool FX, bool FW>
__device__ __forceinline__ void consume(const Args& a, const Quant& qx, const Quant& qw,
                                        uint8_t* tiles, uint64_t* full, uint64_t* empty,
                                        uint8_t* cbuf, Stat& sx, Stat& sw) {
  constexpr int kRow = Tr<T>::kRow;
  const uint32_t bitmap = BM ? uint32_t(BM) : a.bitmap;
  const int rank = BM ? __builtin_popcount(uint32_t(BM)) : a.rank;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  StepIter it;
  it.item = blockIdx.x;
  it.start(a);
  int slot = 0;
  uint32_t phase = 0;
  while (it.item < a.items) {
    ptx::mbar_wait(&full[slot], phase);
    const uint32_t tile = ptx::smem_u32(tiles) + slot * (16 * kRow);
    const int rvalid = a.rows - it.blk * 16;  // rows of this block inside the segment
    // ---------------- phase 1: (row, 16-col block) pieces -> gx operand
    if (GX) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = tid + h * kConsumers;
        const int r = u >> 4, b = u & 15;
        const int c = it.col0 + b * 16;
        if (r < rvalid && c < a.cols) {
          float v[16];
          read16<T>(tile + r * kRow + b * 16 * sizeof(T), v);
          fwht16_raw(v);
          if (MODE == kStats) {
#pragma unroll
            for (int i = 0; i < 16; ++i) sx.add(v[i]);
          } else {
            uint32_t p[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) p[i] = quant2<FX>(make_float2(v[2 * i], v[2 * i + 1]), qx);
            const uint4 out = make_uint4(pack4(p[0], p[1]), pack4(p[2], p[3]), pack4(p[4], p[5]),
                                         pack4(p[6], p[7]));
            const int64_t row = int64_t(it.s) * a.rows + it.blk * 16 + r;
            *reinterpret_cast<uint4*>(a.dst_gx + row * a.ld_gx + c) = out;
          }
        }
      }
    }
    // ---------------- phase 2: column pair -> gw operand (projection along rows)
    if (GW) {
      const int c = 2 * tid;
      if (it.col0 + c < a.cols) {
        float2 pv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (sizeof(T) == 2) {
            const uint32_t w = ptx::lds32(tile + i * kRow + 2 * c);
            pv[i] = make_float2(bf_lo(w), bf_hi(w));
          } else {
            const uint2 w = ptx::lds64(tile + i * kRow + 4 * c);
            pv[i] = make_float2(__uint_as_float(w.x), __uint_as_float(w.y));
          }
        }
        fwht16_pair(pv);
        if (MODE == kStats) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if ((bitmap >> i) & 1u) { sw.add(pv[i].x); sw.add(pv[i].y); }
        } else {
          // codes of kept basis j for both columns, as s16x2 (x = col c, y = col c+1)
          uint32_t cx[4] = {0, 0, 0, 0}, cy[4] = {0, 0, 0, 0};
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if ((bitmap >> i) & 1u) {
              const int j = BM ? __builtin_popcount(uint32_t(BM) & ((1u << i) - 1u))
                               : __popc(bitmap & ((1u << i) - 1u));
              const uint32_t p = quant2<FW>(pv[i], qw);
              const uint32_t bx = (p & 0xFFu) << (8 * (j & 3));
              const uint32_t by = ((p >> 16) & 0xFFu) << (8 * (j & 3));
              switch (j >> 2) {
                case 0: cx[0] |= bx; cy[0] |= by; break;
                case 1: cx[1] |= bx; cy[1] |= by; break;
                case 2: cx[2] |= bx; cy[2] |= by; break;
                default: cx[3] |= bx; cy[3] |= by; break;
              }
            }
          }
          uint8_t* ox = cbuf + c * a.cstride + it.bl * rank;
          uint8_t* oy = ox + a.cstride;
          if (rank == 16) {
            *reinterpret_cast<uint4*>(ox) = make_uint4(cx[0], cx[1], cx[2], cx[3]);
            *reinterpret_cast<uint4*>(oy) = make_uint4(cy[0], cy[1], cy[2], cy[3]);
          } else if (rank == 8) {
            *reinterpret_cast<uint2*>(ox) = make_uint2(cx[0], cx[1]);
            *reinterpret_cast<uint2*>(oy) = make_uint2(cy[0], cy[1]);
          } else if (rank == 4) {
            *reinterpret_cast<uint32_t*>(ox) = cx[0];
            *reinterpret_cast<uint32_t*>(oy) = cy[0];
          } else {
            for (int j = 0; j < rank; ++j) {
              ox[j] = uint8_t(cx[j >> 2] >> (8 * (j & 3)));
              oy[j] = uint8_t(cy[j >> 2] >> (8 * (j & 3)));
            }
          }
        }
      }
    }
    // release the slot to the producer (one arrive per consumer warp)
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[slot]);
    if (++slot == kStages) { slot = 0; phase ^= 1; }
    // ---------------- end of a work item: flush the staged gw codes
    if (GW && MODE == kQuant && it.bl == it.nbl - 1) {
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumers));
      const int run = it.nbl * rank;
      const int64_t k0 = int64_t(it.gb0) * rank;
      const int ncols = min(kCols, a.cols - it.col0);
      if ((run & 15) == 0 && (k0 & 15) == 0) {
        const int chunks = run >> 4;
        for (int i = tid; i < ncols * chunks; i += kConsumers) {
          const int c = i / chunks, q = i - c * chunks;
          *reinterpret_cast<uint4*>(a.dst_gw + (it.col0 + c) * a.ld_gw + k0 + 16 * q) =
              *reinterpret_cast<const uint4*>(cbuf + c * a.cstride + 16 * q);
        }
      } else if ((run & 7) == 0 && (k0 & 7) == 0) {
        const int chunks = run >> 3;
        for (int i = tid; i < ncols * chunks; i += kConsumers) {
          const int c = i / chunks, q = i - c * chunks;
          *reinterpret_cast<uint2*>(a.dst_gw + (it.col0 + c) * a.ld_gw + k0 + 8 * q) =
              *reinterpret_cast<const uint2*>(cbuf + c * a.cstride + 8 * q);
        }
      } else {
        for (int i = tid; i < ncols * run; i += kConsumers) {
          const int c = i / run, q = i - c * run;
          a.dst_gw[(it.col0 + c) * a.ld_gw + k0 + q] = int8_t(cbuf[c * a.cstride + q]);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumers));
    }
    it.next(a);
  }
}

template <typename T, int MODE, bool GX, bool GW, int BM>
__global__ void __launch_bounds__(kThreads) tma_tile_kernel(const __grid_constant__ CUtensorMap map,
                                                           Args a) {
  constexpr int kRow = Tr<T>::kRow;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // pointer arithmetic only (no integer round trip) so the compiler keeps the
  // shared address space and emits LDS/STS rather than generic LD/ST
  uint8_t* tiles = smem_raw + ((128u - (ptx::smem_u32(smem_raw) & 127u)) & 127u);
  uint8_t* cbuf = tiles + kStages * 16 * kRow;
  uint8_t* bars = cbuf + (GW && MODE == kQuant ? kCols * a.cstride : 0);
  bars += (8u - (ptx::smem_u32(bars) & 7u)) & 7u;
  uint64_t* full = reinterpret_cast<uint64_t*>(bars);
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kConsumers / 32);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumers / 32) {
    // ---------------- producer
    if (ptx::elect_one()) {
      ptx::tma_prefetch_desc(&map);
      StepIter it;
      it.item = blockIdx.x;
      it.start(a);
      int slot = 0;
      uint32_t phase = 0;
      while (it.item < a.items) {
        ptx::mbar_wait_sleep(&empty[slot], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[slot], 16 * kRow);
        ptx::tma_load_3d(tiles + slot * 16 * kRow, &map, &full[slot], it.col0, it.blk * 16, it.s);
        if (++slot == kStages) { slot = 0; phase ^= 1; }
        it.next(a);
      }
    }
    return;
  }

  Stat sx, sw;
  if (MODE == kStats) {
    Quant dummy{};
    consume<T, MODE, GX, GW, BM, true, true>(a, dummy, dummy, tiles, full, empty, cbuf, sx, sw);
    sx.warp_reduce();
    sw.warp_reduce();
    if ((threadIdx.x & 31) == 0) {
      if (GX) sx.commit(a.stats);
      if (GW) sw.commit(a.stats + 2);
    }
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
    consume<T, MODE, GX, GW, BM, true, true>(a, qx, qw, tiles, full, empty, cbuf, sx, sw);
  else if (fx)
    consume<T, MODE, GX, GW, BM, true, false>(a, qx, qw, tiles, full, empty, cbuf, sx, sw);
  else if (fw)
    consume<T, MODE, GX, GW, BM, false, true>(a, qx, qw, tiles, full, empty, cbuf, sx, sw);
  else
    consume<T, MODE, GX, GW, BM, false, false>(a, qx, qw, tiles, full, empty, cbuf, sx, sw);
}

template <typename T, int MODE, bool GX, bool GW, int BM>
void launch_one(const CUtensorMap& map, const Args& a, cudaStream_t stream) {
  constexpr int kRow = Tr<T>::kRow;
  const size_t smem = 128 + size_t(kStages) * 16 * kRow +
                      (GW && MODE == kQuant ? size_t(kCols) * a.cstride : 0) + 8 + 2 * kStages * 8;
  auto kern = tma_tile_kernel<T, MODE, GX, GW, BM>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int cap = num_sms() * per_sm;
  const int grid = a.items < 1 ? 1 : (a.items > cap ? cap : a.items);
  kern<<<grid, kThreads, smem, stream>>>(map, a);
}

template <typename T, int MODE, bool GX, bool GW>
void launch_bm(const CUtensorMap& map, const Args& a, cudaStream_t st) {
  if (!GW) return launch_one<T, MODE, GX, GW, 0>(map, a, st);
  switch (a.bitmap) {
    case 0x5555: return launch_one<T, MODE, GX, GW, 0x5555>(map, a, st);  // rank 8 (default plan)
    case 0x1111: return launch_one<T, MODE, GX, GW, 0x1111>(map, a, st);  // rank 4
    case 0x0101: return launch_one<T, MODE, GX, GW, 0x0101>(map, a, st);  // rank 2
    case 0xFFFF: return launch_one<T, MODE, GX, GW, 0xFFFF>(map, a, st);  // full (H.W, rank 16)
    default: return launch_one<T, MODE, GX, GW, 0>(map, a, st);           // calibrated bases
  }
}

template <typename T>
void launch_modes(const CUtensorMap& map, const Args& a, int mode, bool gx, bool gw, cudaStream_t st) {
  if (mode == kStats) {
    if (gx && gw) launch_bm<T, kStats, true, true>(map, a, st);
    else if (gx) launch_bm<T, kStats, true, false>(map, a, st);
    else launch_bm<T, kStats, false, true>(map, a, st);
  } else {
    if (gx && gw) launch_bm<T, kQuant, true, true>(map, a, st);
    else if (gx) launch_bm<T, kQuant, true, false>(map, a, st);
    else launch_bm<T, kQuant, false, true>(map, a, st);
  }
}

// Blocks per work item: >= 32-byte output runs per column when the problem is
// large, while keeping >= ~3 work items per SM.
int choose_nb(int total_blocks, int cols, int rank) {
  int nb = rank >= 8 ? 4 : (rank >= 4 ? 8 : 16);
  const int ncol_tiles = (cols + kCols - 1) / kCols;
  while (nb > 1 && ((total_blocks + nb - 1) / nb) * ncol_tiles < num_sms() * 3) nb >>= 1;
  return nb;
}

}  // namespace

void launch_transform(const TransformArgs& t, int mode, cudaStream_t stream) {
  const size_t esz = t.dtype == kBF16 ? 2 : 4;
  const bool fits32 = t.rows < (int64_t(1) << 30) && t.cols < (int64_t(1) << 30) &&
                      t.segs * ((t.rows + 15) / 16) < (int64_t(1) << 30);
  const bool aligned = (reinterpret_cast<uintptr_t>(t.src) % 16 == 0) && ((t.ld_src * esz) % 16 == 0) &&
                       (t.segs <= 1 || (t.seg_src * esz) % 16 == 0);
  CUtensorMap map;
  bool ok = fits32 && aligned && t.rows > 0 && t.cols > 0 && t.segs > 0;
  if (ok) {
    const uint64_t seg_stride = t.segs > 1 ? uint64_t(t.seg_src) * esz
                                           : (uint64_t(t.rows) * t.ld_src * esz + 15) & ~uint64_t(15);
    const uint64_t dims[3] = {uint64_t(t.cols), uint64_t(t.rows), uint64_t(t.segs)};
    const uint64_t strides[2] = {uint64_t(t.ld_src) * esz, seg_stride};
    const uint32_t box[3] = {uint32_t(kCols), 16, 1};
    ok = encode_tensor_map(&map, t.dtype == kBF16 ? 1 : 2, 3, t.src, dims, strides, box, 0);
  }
  if (!ok) return launch_transform_fallback(t, mode, stream);
  Args a{};
  a.rows = int(t.rows);
  a.cols = int(t.cols);
  a.nblk = int((t.rows + 15) / 16);
  a.total_blocks = int(t.segs) * a.nblk;
  a.rank = t.do_gw ? __builtin_popcount(t.bitmap) : 0;
  a.nb = t.do_gw ? choose_nb(a.total_blocks, a.cols, a.rank) : 4;
  a.ncol_tiles = (a.cols + kCols - 1) / kCols;
  a.items = ((a.total_blocks + a.nb - 1) / a.nb) * a.ncol_tiles;
  a.bitmap = t.bitmap;
  a.bits_gx = t.bits_gx;
  a.bits_gw = t.bits_gw;
  a.stats = t.stats;
  a.dst_gx = t.dst_gx;
  a.ld_gx = t.ld_gx;
  a.dst_gw = t.dst_gw;
  a.ld_gw = t.ld_gw;
  a.scale_gx = t.scale_gx;
  a.scale_gw = t.scale_gw;
  a.cstride = a.nb * a.rank + 16;
  if (t.dtype == kBF16)
    launch_modes<__nv_bfloat16>(map, a, mode, t.do_gx, t.do_gw, stream);
  else
    launch_modes<float>(map, a, mode, t.do_gx, t.do_gw, stream);
}

}  // namespace hlq
