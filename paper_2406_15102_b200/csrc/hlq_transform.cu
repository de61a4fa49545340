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
#include <cstdlib>
#include <atomic>

#include "hlq_b200.h"
#include "hlq_internal.h"
#include "hlq_ptx.cuh"
#include "hlq_quant.cuh"

namespace hlq {

namespace {

using namespace dev;

constexpr int kCols = 256;       // columns per step
constexpr int kConsumers = 128;  // 4 consumer warps
constexpr int kThreads = kConsumers + 32;
#ifndef HLQ_TR_STAGES
#define HLQ_TR_STAGES 4  // 3 / 4 / 5 stages measured within noise (tools/tr_shapes.py)
#endif
constexpr int kStages = HLQ_TR_STAGES;
#ifndef HLQ_TR_MINB
#define HLQ_TR_MINB 4  // CTAs per SM the register budget is sized for
#endif

template <typename T>
struct Tr;
template <>
struct Tr<float> {
  static constexpr int kRow = kCols * 4;
};
template <>
struct Tr<__nv_bfloat16> {
  static constexpr int kRow = kCols * 2;
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
  uint32_t* nonfinite;  // nonfinite_word()
  int pack_gx;          // gx codes as packed int4 (two per byte, low nibble first; ld_gx in bytes)
  int cstride;  // bytes per column in the code staging buffer
#ifdef HLQ_TR_TRACE
  unsigned long long* trace;  // per CTA: 8 globaltimer stamps (development timeline)
#endif
  // conv ACBP (taps > 0): the source is channels-last x read by im2col-mode TMA,
  // one 16-output-pixel block x 256 channels per step and tap; segments =
  // images, rows = output pixels l = ho*Wo + wo, payload row = c*taps + tap
  int taps, kconv, cstr, cpad, wo_n;
  // narrow conv inputs (C = 32 / 64 / 128): tq = 256 / C taps share one step,
  // tap q of the group in columns [q*C, q*C + C) of the tile, stored as tq
  // dense 16 x C sub-tiles (im2col boxes of C channels); tq = 1 otherwise
  int tq, cch;
  // conv ACBP row sharing (stride 1, pad (k-1)/2, Wo % 16 == 0, rank 8): a block of
  // 16 output pixels of row ho and tap (i, j) holds input row ho + i - pad, so tap
  // row i's vectors are tap row `pad`'s vectors shifted by (pad - i) output rows.
  // Only taps [tap0, tap0 + ntap_c) (the middle row) are transformed; the flush
  // writes each block's codes to the other tap rows at the shifted block (zeros
  // where the shifted row falls in the padding).  sh_blk = Wo / 16.
  int tap0, ntap_c, share, sh_blk;
  // row groups (Linear / gy sources with cols = 32 / 64 / 128, taps == 0): a
  // step holds tq = 256 / cols consecutive 16-row blocks as tq dense 16 x cols
  // sub-tiles; items count `vblocks` = ceil(total_blocks / tq) block groups
  int vblocks;
  int cbw;  // columns of the gw staging buffer (cch when row-grouped, else 256)
  int poll_ns;    // grid-barrier polling back-off (HLQ_TR_POLL_NS, development)
  int self_reset; // stats is a library slot: the last CTA to finish zeroes it (kBoth)
  int keep_items; // kBoth: first-pass items loaded evict_last (the second pass's first ones); 0 = no hints
  int dev_flags;  // development A/B (HLQ_TR_FLAGS): 1 = no ticket prefetch, 2 = no grid maxima exchange,
                 // 4 = bias column sums in the QUANT pass (+ a second grid barrier) instead of the STATS pass
  // column sums of the source (the bias gradient), fused into the STATS pass of
  // kBoth: cs_part[g][c] = sum of column c over row group g (one work item's
  // rows), then a fixed-order reduction over g after pass 2 -> cs_out[c]
  float* cs_part;
  float* cs_out;
  int groups;
};

// (item, block) steps of this CTA with 32-bit counters; divisions once per item.
// ord runs over this CTA's ordinals blockIdx.x, +gridDim.x, ...; item = ord, or
// items-1-ord for the reversed second pass of the fused kernel (the last items
// of pass 1 are the ones still in L2 when pass 2 starts).
//
// Dynamic mode (the fused kBoth kernel): each CTA's first item is static
// (blockIdx.x), later ones come from a global ticket counter (ctr) -- CTAs
// sharing an SM, L2 hit rates and the item count per CTA all vary, and a
// static split left the slowest CTA 25 % behind the median in each pass --
// and the producer tells the consumers which (item, block) each ring slot
// holds (at()).
constexpr int kMetaWords = 6;  // per ring slot: col0, s, blk, gb0, nbl | bl << 8 | tap << 16, grp

struct StepIter {
  int ord, item, bl, nbl, gb0, col0, s, blk, tap, grp, ntq;
  int nxt;  // dynamic: the ticket already taken for the next item (fetched one item ahead,
            // so the producer never waits on the atomic's round trip between items)
  bool rev, pf;
  uint32_t* ctr;  // non-null: dynamic tickets
  __device__ __forceinline__ void begin(const Args& a, bool reverse, uint32_t* ticket_ctr = nullptr) {
    rev = reverse;
    ctr = ticket_ctr;
    ord = int(blockIdx.x);  // first item static (a greedy first grab let early CTAs queue two)
    // prefetching pays with many items per CTA; with ~2 it lengthens the tail
    pf = ctr && a.items >= 4 * int(gridDim.x) && !(a.dev_flags & 1);
    if (pf && ord < a.items) nxt = int(gridDim.x + atomicAdd(ctr, 1u));
    start(a);
  }
  __device__ __forceinline__ void setup(const Args& a, int i) {
    item = i;
    int rest = item;
    tap = 0;
    ntq = 1;
    if (a.taps) {  // tap groups innermost: concurrent CTAs reuse the same x pixels through L2
      const int ntg = (a.ntap_c + a.tq - 1) / a.tq;
      rest = item / ntg;
      tap = a.tap0 + (item - rest * ntg) * a.tq;
      ntq = min(a.tq, a.tap0 + a.ntap_c - tap);
    }
    const int g = rest / a.ncol_tiles;
    grp = g;
    col0 = (rest - g * a.ncol_tiles) * kCols;
    gb0 = g * a.nb;
    nbl = min(a.nb, a.vblocks - gb0);
  }
  // producer -> consumers: everything a step needs, so the consumers do no
  // integer divisions (they were ~25 % of the ACBP kernel's instructions)
  __device__ __forceinline__ void publish(int* m) const {
    m[0] = col0; m[1] = s; m[2] = blk; m[3] = gb0; m[4] = nbl | (bl << 8) | (tap << 16) | (ntq << 24); m[5] = grp;
  }
  __device__ __forceinline__ void load(const volatile int* m) {
    col0 = m[0]; s = m[1]; blk = m[2]; gb0 = m[3];
    const int pk = m[4];
    nbl = pk & 0xFF; bl = (pk >> 8) & 0xFF; tap = (pk >> 16) & 0xFF; ntq = (pk >> 24) & 0xFF;
    grp = m[5];
  }
  __device__ __forceinline__ bool valid(const Args& a) const { return ord < a.items; }
  __device__ __forceinline__ void start(const Args& a) {
    if (ord >= a.items) return;
    setup(a, rev ? a.items - 1 - ord : ord);
    bl = 0;
    s = gb0 / a.nblk;
    blk = gb0 - s * a.nblk;
  }
  __device__ __forceinline__ void next(const Args& a) {
    if (++bl == nbl) {
      if (pf) {
        ord = nxt;
        if (ord < a.items) nxt = int(gridDim.x + atomicAdd(ctr, 1u));
      } else if (ctr) {
        ord = int(gridDim.x + atomicAdd(ctr, 1u));
      } else {
        ord += int(gridDim.x);
      }
      start(a);
    } else if (++blk == a.nblk) {
      blk = 0;
      ++s;
    }
  }
};

// bf16 row pieces: the 8 words (2 columns each) of rows A and B
__device__ __forceinline__ void load16x2_bf16(uint32_t pa, uint32_t pb, uint32_t (&wa)[8], uint32_t (&wb)[8]) {
  const uint4 ta[2] = {ptx::lds128(pa), ptx::lds128(pa + 16)};
  const uint4 tb[2] = {ptx::lds128(pb), ptx::lds128(pb + 16)};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    wa[4 * q] = ta[q].x; wa[4 * q + 1] = ta[q].y; wa[4 * q + 2] = ta[q].z; wa[4 * q + 3] = ta[q].w;
    wb[4 * q] = tb[q].x; wb[4 * q + 1] = tb[q].y; wb[4 * q + 2] = tb[q].z; wb[4 * q + 3] = tb[q].w;
  }
}
__device__ __forceinline__ void unpack16x2_bf16(const uint32_t (&wa)[8], const uint32_t (&wb)[8], float2 (&p)[16]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    p[2 * k] = make_float2(bf_lo(wa[k]), bf_lo(wb[k]));
    p[2 * k + 1] = make_float2(bf_hi(wa[k]), bf_hi(wb[k]));
  }
}

// Two 16-element row pieces (rows r and r+8 of the staged tile, same column
// block) as 16 f32x2 lanes: p[i] = (A[i], B[i]).  All four butterfly stages
// then run on packed pairs.
template <typename T>
__device__ __forceinline__ void read16x2(uint32_t pa, uint32_t pb, float2 (&p)[16], uint32_t flip) {
  if (sizeof(T) == 2) {
    (void)flip;  // swapping the halves per thread costs more SELs than the 2-way conflict
    uint32_t wa[8], wb[8];
    load16x2_bf16(pa, pb, wa, wb);
    unpack16x2_bf16(wa, wb, p);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 ta = ptx::lds128(pa + 16 * q), tb = ptx::lds128(pb + 16 * q);
      p[4 * q] = make_float2(__uint_as_float(ta.x), __uint_as_float(tb.x));
      p[4 * q + 1] = make_float2(__uint_as_float(ta.y), __uint_as_float(tb.y));
      p[4 * q + 2] = make_float2(__uint_as_float(ta.z), __uint_as_float(tb.z));
      p[4 * q + 3] = make_float2(__uint_as_float(ta.w), __uint_as_float(tb.w));
    }
  }
}

// Conv ACBP row sharing (Args::share): the rank-8 codes of block gb of payload
// row pr (tap (pad, j), channel c) are also the codes of tap (i, j) at the block
// (pad - i) output rows further (same image); rows whose source would be the
// padding get zeros, written by the block of the same output row.
__device__ __forceinline__ void share_copy(const Args& a, int64_t pr, int gb, uint2 v) {
  const int img = gb / a.nblk, lb = gb - img * a.nblk;
  const int ho = lb / a.sh_blk, ho_n = a.rows / (16 * a.sh_blk);  // output rows per image
  const int pad = a.tap0 / a.kconv;
  for (int i = 0; i < a.kconv; ++i) {
    if (i == pad) continue;
    const int64_t row = pr + int64_t(i - pad) * a.kconv;
    const int hd = ho + (pad - i);  // destination output row holding this vector
    if (hd >= 0 && hd < ho_n)
      *reinterpret_cast<uint2*>(a.dst_gw + row * a.ld_gw + int64_t(gb + (pad - i) * a.sh_blk) * 8) = v;
    // the destination row ho of tap row i whose source row lies in the padding
    const int src = ho + i - pad;
    if (src < 0 || src >= ho_n)
      *reinterpret_cast<uint2*>(a.dst_gw + row * a.ld_gw + int64_t(gb) * 8) = make_uint2(0u, 0u);
  }
}

template <typename T, int MODE, bool GX, bool GW, int BM, bool FX, bool FW, bool DYN, int GRP>
__device__ __forceinline__ void consume(const Args& a, const Quant& qx, const Quant& qw,
                                        uint8_t* tiles, uint64_t* full, uint64_t* empty,
                                        const volatile int* meta, uint8_t* cbuf, Stat& sx, Stat& sw,
                                        int& slot, uint32_t& phase, bool reverse, uint32_t* shmax = nullptr) {
  constexpr int kRow = Tr<T>::kRow;
  const uint32_t bitmap = BM ? uint32_t(BM) : a.bitmap;
  const int rank = BM ? __builtin_popcount(uint32_t(BM)) : a.rank;
  const int tid = threadIdx.x;
  const int lane = threadIdx.x & 31;
  constexpr bool p1 = true, p2 = true;
  const int ftid = tid;
  constexpr int kFlushThreads = kConsumers;
  StepIter it;
  if (!DYN) it.begin(a, reverse);
  float2 csum = make_float2(0.0f, 0.0f);
  // bf16 STATS pass: L1-bound block skipping + min nonzero from the inputs
  // (hlq_quant.cuh, "bound statistics"); fp32 sources keep the exact pass
#ifdef HLQ_TR_EXACT_STATS
  constexpr bool kBound = false;
#else
  constexpr bool kBound = MODE == kStats && sizeof(T) == 2;
#endif
  // the bias column sums run in the STATS pass (partials ready at the grid
  // barrier) unless dev flag 4 moves them to the QUANT pass
  const bool cs_here = a.cs_part && (MODE == ((a.dev_flags & 4) ? kQuant : kStats));
  uint32_t mz = 0x7FFF7FFFu;      // running s16x2 min of |x| bits + 0x7FFF
  float thr_x = 0.0f, thr_w = 0.0f;  // skip thresholds from the running exact maxima
  // per-thread tile geometry, fixed for the whole launch (hoisted: the grouped
  // variants had spent a signed integer division per thread and step on it)
  const int g1_q = GRP == 2 ? (tid & 15) / (a.cch >> 4) : 0;    // phase 1, row groups: sub-tile
  const int g1_bb = GRP == 2 ? (tid & 15) - g1_q * (a.cch >> 4) : (tid & 15);
  const int g2_q = GRP ? (2 * tid) / a.cch : 0;                  // phase 2: sub-tile of column 2*tid
  const int g2_cc = 2 * tid - g2_q * (GRP ? a.cch : 0);
  const uint32_t g2_pitch = GRP ? uint32_t(a.cch) * sizeof(T) : uint32_t(kRow);
  const uint32_t g2_off = GRP ? uint32_t(g2_q) * 16u * g2_pitch + uint32_t(g2_cc) * sizeof(T)
                              : uint32_t(2 * tid) * sizeof(T);
  while (DYN || it.valid(a)) {
    {
      ptx::mbar_wait(&full[slot], phase);
      if (DYN) {
        const volatile int* m = meta + kMetaWords * slot;
        if (m[0] < 0) {  // the producer found no more items for this pass
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&empty[slot]);
          if (++slot == kStages) { slot = 0; phase ^= 1; }
          break;
        }
        it.load(m);
      }
      const uint32_t tile = ptx::smem_u32(tiles) + slot * (16 * kRow);
      constexpr bool rg = GRP == 2;  // row-grouped narrow source (GRP 1: conv tap groups)
      // running maxima shared by the CTA's warps and, through the producer
      // (once per work item), with the grid (hlq_quant.cuh bound statistics)
      uint2 gmax = make_uint2(0u, 0u);
      if (kBound) gmax = ptx::lds64(ptx::smem_u32(shmax));
      if (rg && !DYN) {  // static schedule: the first real block of this step (dynamic: published)
        const int rb = (it.gb0 + it.bl) * a.tq;
        it.s = rb / a.nblk;
        it.blk = rb - it.s * a.nblk;
      }
      const int rb0 = (it.gb0 + it.bl) * a.tq;  // rg: first real block of the step
      const int rvalid = a.rows - it.blk * 16;  // rows of this block inside the segment
      // ---------------- phase 1: (row, 16-col block) pieces -> gx operand
      // thread = (rows r and r+8, block b); rows past the segment and columns
      // past `cols` were zero-filled by TMA, so the statistics need no predicate
      if (GX && p1) {
        const int r = tid >> 4, b = tid & 15;
        // rg: 16-col block b is block bb of sub-tile q (real block rb0 + q)
        int bb = b, ps = it.s, pb = it.blk, prv = rvalid;
        uint32_t pitch = kRow, base = tile;
        bool ok = true;
        if (rg) {
          const int q = g1_q;
          bb = g1_bb;
          pitch = uint32_t(a.cch) * sizeof(T);
          base = tile + q * 16 * pitch;
          ok = rb0 + q < a.total_blocks;
          pb += q;
          while (pb >= a.nblk) { pb -= a.nblk; ++ps; }
          prv = a.rows - pb * 16;
        }
        const int c = it.col0 + bb * 16;
        if (kBound) {
          uint32_t wa[8], wb[8];
          if (ok) {
            load16x2_bf16(base + r * pitch + bb * 16 * sizeof(T), base + (r + 8) * pitch + bb * 16 * sizeof(T), wa,
                          wb);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) wa[k] = wb[k] = 0u;
          }
          uint32_t aa[8], ab[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            aa[k] = wa[k] & kAbs2;
            ab[k] = wb[k] & kAbs2;
            mz = s16x2_min3(mz, aa[k] + kAbs2, ab[k] + kAbs2);
          }
          const uint32_t sA = bf2_tree<8>(aa), sB = bf2_tree<8>(ab);
          const uint32_t l1 = bf2_add(__byte_perm(sA, sB, 0x5410), __byte_perm(sA, sB, 0x7632));  // (L1 A, L1 B)
          const bool need = !(bf2_lane_max(l1) <= thr_x);
          if (need) {
            float2 p[16];
            unpack16x2_bf16(wa, wb, p);
            fwht16_pair(p);
#pragma unroll
            for (int i = 0; i < 16; ++i) sx.amax2(p[i].x, p[i].y);
          }
          // share the best maximum across the warp and the grid (any exact block
          // maximum bounds the result; NaN bits 0x7FFFFFFF win the max and stop skipping)
          if (__any_sync(0xffffffffu, need)) {
            const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(sx.amax) & 0x7FFFFFFFu);
            if (lane == 0 && wm > gmax.x) atomicMax(shmax, wm);
            thr_x = fmaxf(thr_x, bound_thr(__uint_as_float(wm)));
          }
          thr_x = fmaxf(thr_x, bound_thr(__uint_as_float(gmax.x)));
        } else {
        float2 p[16];
        if (ok)
          read16x2<T>(base + r * pitch + bb * 16 * sizeof(T), base + (r + 8) * pitch + bb * 16 * sizeof(T), p,
                      uint32_t(b >> 2) & 1u);
        else
#pragma unroll
          for (int i = 0; i < 16; ++i) p[i] = make_float2(0.0f, 0.0f);
        fwht16_pair(p);
        if (MODE == kStats) {
#pragma unroll
          for (int i = 0; i < 16; ++i) sx.add2(p[i].x, p[i].y);
        } else if (ok && c < a.cols) {
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) w[i] = quant2<FX>(p[i], qx);  // (code A_i, code B_i)
          uint32_t ca[4], cb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t t01 = __byte_perm(w[4 * q], w[4 * q + 1], 0x6420);  // A B A B
            const uint32_t t23 = __byte_perm(w[4 * q + 2], w[4 * q + 3], 0x6420);
            ca[q] = __byte_perm(t01, t23, 0x6420);
            cb[q] = __byte_perm(t01, t23, 0x7531);
          }
          const int64_t row = int64_t(ps) * a.rows + pb * 16 + r;
          if (a.pack_gx) {
            // nibble pairs: n_j = codes (2j, 2j+1) of row A in byte 0, of row B in byte 2
            // (the ACBP container's nibble order, low nibble first, acbp.py:56-61)
            uint32_t n[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t hi = w[2 * j + 1] << 4;
              asm("lop3.b32 %0, %1, %2, 0x000F000F, 0xE4;" : "=r"(n[j]) : "r"(w[2 * j]), "r"(hi));  // (a & c) | (b & ~c)
            }
            uint32_t pa[2], pb2[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t t01 = __byte_perm(n[4 * q], n[4 * q + 1], 0x6420);
              const uint32_t t23 = __byte_perm(n[4 * q + 2], n[4 * q + 3], 0x6420);
              pa[q] = __byte_perm(t01, t23, 0x6420);
              pb2[q] = __byte_perm(t01, t23, 0x7531);
            }
            if (r < prv) *reinterpret_cast<uint2*>(a.dst_gx + row * a.ld_gx + (c >> 1)) = make_uint2(pa[0], pa[1]);
            if (r + 8 < prv)
              *reinterpret_cast<uint2*>(a.dst_gx + (row + 8) * a.ld_gx + (c >> 1)) = make_uint2(pb2[0], pb2[1]);
          } else {
            if (r < prv)
              *reinterpret_cast<uint4*>(a.dst_gx + row * a.ld_gx + c) = make_uint4(ca[0], ca[1], ca[2], ca[3]);
            if (r + 8 < prv)
              *reinterpret_cast<uint4*>(a.dst_gx + (row + 8) * a.ld_gx + c) =
                  make_uint4(cb[0], cb[1], cb[2], cb[3]);
          }
        }
        }  // !kBound
      }
      // ---------------- phase 2: column pair -> gw operand (projection along rows)
      if (GW && p2) {
        const int c = 2 * tid;
        // tap-grouped (conv) tiles: column c is channel c % cch of tap (tap + c / cch);
        // row-grouped tiles: column c % cch of real block rb0 + c / cch
        const int q = g2_q;
        const int cc = g2_cc;  // source column inside the sub-tile (== c when tq == 1)
        const uint32_t pitch = g2_pitch;
        const uint32_t col_addr = tile + g2_off;
        const bool in = GRP == 0 ? it.col0 + c < a.cols : (rg ? rb0 + q < a.total_blocks : q < it.ntq);
        bool need_w = false;
        if (kBound && in) {
          uint32_t w[16], av[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            w[i] = ptx::lds32(col_addr + i * pitch);
            av[i] = w[i] & kAbs2;
          }
          if (!GX) {  // no phase 1 to take the input minimum
#pragma unroll
            for (int i = 0; i < 8; ++i) mz = s16x2_min3(mz, av[2 * i] + kAbs2, av[2 * i + 1] + kAbs2);
          }
          // (conv rows past the image, zeroed below, only loosen the bound)
          need_w = !(bf2_lane_max(bf2_tree<16>(av)) <= thr_w);
          if (cs_here) {
            // bias column sums: the pairwise tree in the butterfly's DC order (stages
            // h = 1, 2, 4, 8), accumulated over the item's blocks
            float2 t[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              t[i] = f2add(make_float2(bf_lo(w[2 * i]), bf_hi(w[2 * i])),
                           make_float2(bf_lo(w[2 * i + 1]), bf_hi(w[2 * i + 1])));
#pragma unroll
            for (int i = 0; i < 4; ++i) t[i] = f2add(t[2 * i], t[2 * i + 1]);
            const float2 blk_sum = f2add(f2add(t[0], t[1]), f2add(t[2], t[3]));
            csum = it.bl == 0 ? blk_sum : f2add(csum, blk_sum);
            if (it.bl == it.nbl - 1) {
              const int oc = rg ? cc : it.col0 + c;
              float* o = a.cs_part + int64_t(oc) * a.groups + (rg ? it.grp * a.tq + q : it.grp);
              o[0] = csum.x;
              if (oc + 1 < a.cols) o[a.groups] = csum.y;
            }
          }
          if (need_w) {
            float2 pv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pv[i] = make_float2(bf_lo(w[i]), bf_hi(w[i]));
            if (a.taps && rvalid < 16) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i >= rvalid) pv[i] = make_float2(0.0f, 0.0f);
            }
            fwht16_pair(pv);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if ((bitmap >> i) & 1u) sw.amax2(pv[i].x, pv[i].y);
          }
        } else if (in) {
          float2 pv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (sizeof(T) == 2) {
              const uint32_t w = ptx::lds32(col_addr + i * pitch);
              pv[i] = make_float2(bf_lo(w), bf_hi(w));
            } else {
              const uint2 w = ptx::lds64(col_addr + i * pitch);
              pv[i] = make_float2(__uint_as_float(w.x), __uint_as_float(w.y));
            }
          }
          // conv: the im2col walk runs on into the next image after the last
          // pixel of this one; the reference zero-pads L (tensor.py:125-135)
          if (a.taps && rvalid < 16) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i >= rvalid) pv[i] = make_float2(0.0f, 0.0f);
          }
          // column sums of the 16 rows, accumulated over the item (the bias gradient):
          // the un-normalised DC coefficient of the projection butterfly IS the pairwise
          // tree ((x0+x1)+(x2+x3))+... in the same order (stages h = 1, 2, 4, 8), so
          // when basis 0 is kept the sum comes for free from pv[0]; otherwise the tree
          const bool dc_kept = (bitmap & 1u) != 0;
          float2 blk_sum = make_float2(0.0f, 0.0f);
          if (cs_here && !dc_kept) {
            float2 t[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) t[i] = f2add(pv[2 * i], pv[2 * i + 1]);
#pragma unroll
            for (int i = 0; i < 4; ++i) t[i] = f2add(t[2 * i], t[2 * i + 1]);
            blk_sum = f2add(f2add(t[0], t[1]), f2add(t[2], t[3]));
          }
          fwht16_pair(pv);
          // (kQuant: the fused kernel's second pass; its partials are reduced
          // after a second grid barrier)
          if (cs_here) {
            if (dc_kept) blk_sum = pv[0];
            csum = it.bl == 0 ? blk_sum : f2add(csum, blk_sum);
            if (it.bl == it.nbl - 1) {
              // column-major partials: a column's groups are contiguous for the final sum
              // (rg: one partial per sub-tile position q of the item's steps)
              const int oc = rg ? cc : it.col0 + c;
              float* o = a.cs_part + int64_t(oc) * a.groups + (rg ? it.grp * a.tq + q : it.grp);
              o[0] = csum.x;
              if (oc + 1 < a.cols) o[a.groups] = csum.y;
            }
          }
          if (MODE == kStats) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if ((bitmap >> i) & 1u) sw.add2(pv[i].x, pv[i].y);
          } else {
            // codes of kept basis j for both columns, as s16x2 (x = col c, y = col c+1)
            uint32_t cx[4] = {0, 0, 0, 0}, cy[4] = {0, 0, 0, 0};
            constexpr int kRankC = BM ? __builtin_popcount(uint32_t(BM)) : 0;
            if (BM && (kRankC & 3) == 0) {
              // compile-time bases, rank 4/8/16: byte-pack 4 codes per column with 4 PRMTs
              uint32_t w[16];
              int j = 0;
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if ((uint32_t(BM) >> i) & 1u) w[j++] = quant2<FW>(pv[i], qw);
#pragma unroll
              for (int g = 0; g < kRankC / 4; ++g) {
                const uint32_t t01 = __byte_perm(w[4 * g], w[4 * g + 1], 0x6420);
                const uint32_t t23 = __byte_perm(w[4 * g + 2], w[4 * g + 3], 0x6420);
                cx[g] = __byte_perm(t01, t23, 0x6420);
                cy[g] = __byte_perm(t01, t23, 0x7531);
              }
            } else {
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
            }
            // staged in smem, flushed per item as K-major runs (direct 8-byte
            // global stores measured slower: 94 vs 80 us on the fc2-input ACBP)
            uint8_t* ox = rg ? cbuf + cc * a.cstride + (it.bl * a.tq + q) * rank : cbuf + c * a.cstride + it.bl * rank;
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
        } else if (cs_here && rg) {
          // a sub-tile past the last real block: its column sums still need the
          // item's partial written (zero when the item had no other step)
          if (it.bl == 0) csum = make_float2(0.0f, 0.0f);
          if (it.bl == it.nbl - 1) {
            float* o = a.cs_part + int64_t(cc) * a.groups + it.grp * a.tq + q;
            o[0] = csum.x;
            if (cc + 1 < a.cols) o[a.groups] = csum.y;
          }
        }
        if (kBound) {
          if (__any_sync(0xffffffffu, need_w)) {
            const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(sw.amax) & 0x7FFFFFFFu);
            if (lane == 0 && wm > gmax.y) atomicMax(shmax + 1, wm);
            thr_w = fmaxf(thr_w, bound_thr(__uint_as_float(wm)));
          }
          thr_w = fmaxf(thr_w, bound_thr(__uint_as_float(gmax.y)));
        }
      }
      // release the slot to the producer (one arrive per consuming warp)
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[slot]);
    }
    if (++slot == kStages) { slot = 0; phase ^= 1; }
    // ---------------- end of a work item: flush the staged gw codes
    if (GW && MODE == kQuant && it.bl == it.nbl - 1) {
      asm volatile("bar.sync 1, %0;" ::"n"(kFlushThreads));
      constexpr bool rgf = GRP == 2;
      const int run = rgf ? (min(a.total_blocks, (it.gb0 + it.nbl) * a.tq) - it.gb0 * a.tq) * rank : it.nbl * rank;
      const int64_t k0 = int64_t(rgf ? it.gb0 * a.tq : it.gb0) * rank;
      const int orow = a.taps ? a.taps : 1;  // payload row of column c: c (Linear) or c*taps + tap (conv)
      const int ncols = rgf ? a.cch : (GRP == 1 ? it.ntq * a.cch : min(kCols, a.cols - it.col0));
      // payload row of tile column c (tap-grouped: channel c % cch, tap + c / cch)
      // (cch of a tap-grouped tile is 32 / 64 / 128: shifts, not divisions)
      const int csh = __ffs(GRP == 1 ? a.cch : 1) - 1;
      auto prow = [&](int c) -> int64_t {
        if (GRP == 1) {
          const int qq = c >> csh;
          return int64_t(c - (qq << csh)) * orow + it.tap + qq;
        }
        return int64_t(it.col0 + c) * orow + it.tap;
      };
      if ((run & 15) == 0 && (k0 & 15) == 0) {
        const int chunks = run >> 4;
        const int chsh = __ffs(chunks) - 1;  // chunks = nbl * rank / 16 (rank 8 / 16, nbl a power of two)
        const bool chpow2 = (chunks & (chunks - 1)) == 0;
        for (int i = ftid; i < ncols * chunks; i += kFlushThreads) {
          const int c = chpow2 ? (i >> chsh) : i / chunks, q = i - c * chunks;
          const uint4 v = *reinterpret_cast<const uint4*>(cbuf + c * a.cstride + 16 * q);
          const int64_t pr = prow(c);
          *reinterpret_cast<uint4*>(a.dst_gw + pr * a.ld_gw + k0 + 16 * q) = v;
          if (a.share) {
            share_copy(a, pr, it.gb0 + 2 * q, make_uint2(v.x, v.y));
            share_copy(a, pr, it.gb0 + 2 * q + 1, make_uint2(v.z, v.w));
          }
        }
      } else if ((run & 7) == 0 && (k0 & 7) == 0) {
        const int chunks = run >> 3;
        for (int i = ftid; i < ncols * chunks; i += kFlushThreads) {
          const int c = i / chunks, q = i - c * chunks;
          const uint2 v = *reinterpret_cast<const uint2*>(cbuf + c * a.cstride + 8 * q);
          const int64_t pr = prow(c);
          *reinterpret_cast<uint2*>(a.dst_gw + pr * a.ld_gw + k0 + 8 * q) = v;
          if (a.share) share_copy(a, pr, it.gb0 + q, v);
        }
      } else {
        for (int i = ftid; i < ncols * run; i += kFlushThreads) {
          const int c = i / run, q = i - c * run;
          a.dst_gw[prow(c) * a.ld_gw + k0 + q] = int8_t(cbuf[c * a.cstride + q]);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kFlushThreads));
    }
    if (!DYN) it.next(a);
  }
  if (kBound) {  // both operands are transforms of the same inputs: one lower bound
    const float mnz = mz_to_mnz(mz);
    sx.mnz = mnz;
    sw.mnz = mnz;
  }
}

// Quant-pass dispatch on the (grid-uniform) fast-division guard of each operand.
template <typename T, bool GX, bool GW, int BM, bool DYN, int GRP>
__device__ __forceinline__ void consume_quant(const Args& a, uint8_t* tiles, uint64_t* full,
                                              uint64_t* empty, const volatile int* meta, uint8_t* cbuf,
                                              int& slot, uint32_t& phase, bool reverse) {
  Quant qx{}, qw{};
  if (GX) qx = make_quant(a.stats, a.bits_gx);
  if (GW) qw = make_quant(a.stats + 2, a.bits_gw);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (GX && a.scale_gx) *a.scale_gx = qx.s;
    if (GW && a.scale_gw) *a.scale_gw = qw.s;
    if (GX) flag_nonfinite(qx, a.nonfinite);
    if (GW) flag_nonfinite(qw, a.nonfinite);
  }
  Stat sx, sw;
  const bool fx = !GX || qx.fast, fw = !GW || qw.fast;
  if (fx && fw)
    consume<T, kQuant, GX, GW, BM, true, true, DYN, GRP>(a, qx, qw, tiles, full, empty, meta, cbuf, sx, sw, slot, phase,
                                                   reverse);
  else if (fx)
    consume<T, kQuant, GX, GW, BM, true, false, DYN, GRP>(a, qx, qw, tiles, full, empty, meta, cbuf, sx, sw, slot, phase,
                                                   reverse);
  else if (fw)
    consume<T, kQuant, GX, GW, BM, false, true, DYN, GRP>(a, qx, qw, tiles, full, empty, meta, cbuf, sx, sw, slot, phase,
                                                   reverse);
  else
    consume<T, kQuant, GX, GW, BM, false, false, DYN, GRP>(a, qx, qw, tiles, full, empty, meta, cbuf, sx, sw, slot, phase,
                                                   reverse);
}

// Grid-wide barrier among the consumer warps of co-resident CTAs (cooperative
// launch): thread 0 publishes this CTA's arrival with a release reduction (no
// returned value to wait for), after the CTA's prior writes were collected by
// the named barrier, and polls with acquire loads until `target` arrivals.
__device__ __forceinline__ void grid_barrier(uint32_t* ctr, uint32_t target, int poll_ns) {
  if (threadIdx.x == 0) {
    uint32_t seen = 0;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
    while (seen < target) {
      // every CTA polls the same L2 line: back off so the arrivals and the
      // statistics reductions queued on that slice are not delayed
      __nanosleep(poll_ns);
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
    }
  }
  asm volatile("bar.sync 2, %0;" ::"n"(kConsumers) : "memory");
}

// MODE kStats / kQuant: one pass.  MODE kBoth: both passes in one cooperative
// launch -- statistics, a grid-wide barrier (a counter in stats[32]), then the
// quantization pass over the items in reverse order.  The producer warp never
// waits for the barrier: it keeps streaming pass-2 tiles into the ring while
// the consumers wait for the scales.
template <typename T, int MODE, bool GX, bool GW, int BM, int GRP>
__global__ void __launch_bounds__(kThreads, HLQ_TR_MINB) tma_tile_kernel(const __grid_constant__ CUtensorMap map,
                                                           Args a) {
  constexpr int kRow = Tr<T>::kRow;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // pointer arithmetic only (no integer round trip) so the compiler keeps the
  // shared address space and emits LDS/STS rather than generic LD/ST
  uint8_t* tiles = smem_raw + ((128u - (ptx::smem_u32(smem_raw) & 127u)) & 127u);
  uint8_t* cbuf = tiles + kStages * 16 * kRow;
  uint8_t* bars = cbuf + (GW && MODE != kStats ? a.cbw * a.cstride : 0);
  bars += (8u - (ptx::smem_u32(bars) & 7u)) & 7u;
  uint64_t* full = reinterpret_cast<uint64_t*>(bars);
  uint64_t* empty = full + kStages;
  int* meta = reinterpret_cast<int*>(empty + kStages);  // dynamic mode: kMetaWords per slot
  uint32_t* shmax = reinterpret_cast<uint32_t*>(meta + kStages * kMetaWords);  // bound stats: CTA maxima (x, w)
  constexpr bool kBoundK = (MODE == kStats || MODE == kBoth) && sizeof(T) == 2;
#ifdef HLQ_TR_STATIC
  constexpr bool kDyn = false;  // A/B builds
#else
  constexpr bool kDyn = MODE == kBoth;
#endif

  const int warp = threadIdx.x >> 5;
#ifdef HLQ_TR_TRACE
  auto stamp = [&](int i) {
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[blockIdx.x * 8 + i] = t;
    }
  };
#else
  auto stamp = [](int) {};
#endif
  stamp(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kConsumers / 32);
    }
    shmax[0] = shmax[1] = 0u;
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // programmatic dependent launch: the source (and everything else) is read
  // only after the previous kernel on the stream has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == kConsumers / 32) {
    // ---------------- producer
    if (ptx::elect_one()) {
      ptx::tma_prefetch_desc(&map);
      const uint64_t pol_last = ptx::createpolicy_evict_last(), pol_first = ptx::createpolicy_evict_first();
      int slot = 0;
      uint32_t phase = 0;
      for (int pass = 0; pass < (MODE == kBoth ? 2 : 1); ++pass) {
        StepIter it;
        it.begin(a, pass == 1, kDyn ? a.stats + 64 + 32 * pass : nullptr);
        uint4 gpend = make_uint4(0u, 0u, 0u, 0u);  // the grid maxima loaded at the previous item
        while (it.valid(a)) {
          if (kBoundK && pass == 0 && it.bl == 0 && !(a.dev_flags & 2)) {
            // fold the grid's maxima into the CTA's, publish the CTA's (one relaxed
            // load and at most two reductions per item: no same-line hot spot)
            const uint32_t cx = *reinterpret_cast<volatile uint32_t*>(shmax);
            const uint32_t cw = *reinterpret_cast<volatile uint32_t*>(shmax + 1);
            if (GX && cx > gpend.x) asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(a.stats), "r"(cx) : "memory");
            if (GW && cw > gpend.z) asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(a.stats + 2), "r"(cw) : "memory");
            if (gpend.x > cx) atomicMax(shmax, gpend.x);
            if (gpend.z > cw) atomicMax(shmax + 1, gpend.z);
            asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(gpend.x), "=r"(gpend.y), "=r"(gpend.z), "=r"(gpend.w) : "l"(a.stats));
          }
          ptx::mbar_wait_sleep(&empty[slot], phase ^ 1);
          constexpr bool rgp = GRP == 2;
          if (rgp) {  // first real block of this step's group
            const int rb = (it.gb0 + it.bl) * a.tq;
            it.s = rb / a.nblk;
            it.blk = rb - it.s * a.nblk;
          }
          if (kDyn) it.publish(meta + kMetaWords * slot);
          if (a.taps) {
            const int l0 = it.blk * 16, ho = l0 / a.wo_n, wo = l0 - ho * a.wo_n;
            const uint32_t sub = GRP == 1 ? uint32_t(16 * a.cch * sizeof(T)) : uint32_t(16 * kRow);
            ptx::mbar_arrive_expect_tx(&full[slot], sub * uint32_t(it.ntq));
            int ti = it.tap / a.kconv, tj = it.tap - ti * a.kconv;  // one division per step
            for (int q = 0; q < it.ntq; ++q) {
              ptx::tma_load_im2col_4d(tiles + slot * 16 * kRow + q * sub, &map, &full[slot], it.col0,
                                      wo * a.cstr - a.cpad, ho * a.cstr - a.cpad, it.s, uint16_t(tj),
                                      uint16_t(ti));
              if (++tj == a.kconv) { tj = 0; ++ti; }
            }
          } else if (rgp) {
            const int rb = (it.gb0 + it.bl) * a.tq;
            const int nv = min(a.tq, a.total_blocks - rb);
            const uint32_t sub = uint32_t(16 * a.cch * sizeof(T));
            ptx::mbar_arrive_expect_tx(&full[slot], sub * uint32_t(nv));
            int ps = it.s, pb = it.blk;
            for (int q = 0; q < nv; ++q) {
              ptx::tma_load_3d(tiles + slot * 16 * kRow + q * sub, &map, &full[slot], 0, pb * 16, ps);
              if (++pb == a.nblk) { pb = 0; ++ps; }
            }
          } else {
            ptx::mbar_arrive_expect_tx(&full[slot], 16 * kRow);
            if (MODE == kBoth && a.keep_items > 0) {
              // L2 residency for the second pass (which walks the items in reverse):
              // the last keep_items of the first pass stay (evict_last), everything
              // else streams through (evict_first)
              const bool keep = pass == 0 && it.ord >= a.items - a.keep_items;
              ptx::tma_load_3d_hint(tiles + slot * 16 * kRow, &map, &full[slot], it.col0, it.blk * 16, it.s,
                                    keep ? pol_last : pol_first);
            } else {
              ptx::tma_load_3d(tiles + slot * 16 * kRow, &map, &full[slot], it.col0, it.blk * 16, it.s);
            }
          }
          if (++slot == kStages) { slot = 0; phase ^= 1; }
          it.next(a);
        }
        if (kDyn) {  // end-of-pass sentinel slot
          ptx::mbar_wait_sleep(&empty[slot], phase ^ 1);
          meta[kMetaWords * slot] = -1;
          ptx::mbar_arrive(&full[slot]);
          if (++slot == kStages) { slot = 0; phase ^= 1; }
        }
      }
    }
    if (MODE == kBoth && a.self_reset) {
      // join the final CTA barrier: this warp's ticket / maxima atomics are then
      // ordered before the CTA's arrival at the slot's done counter
      __syncthreads();
    }
    return;
  }

  int slot = 0;
  uint32_t phase = 0;
  if (MODE == kQuant) {
    consume_quant<T, GX, GW, BM, false, GRP>(a, tiles, full, empty, meta, cbuf, slot, phase, false);
    return;
  }
  Stat sx, sw;
  {
    Quant dummy{};
    consume<T, kStats, GX, GW, BM, true, true, kDyn, GRP>(a, dummy, dummy, tiles, full, empty, meta, cbuf, sx, sw,
                                                     slot, phase, false, shmax);
  }
  stamp(1);
  sx.warp_reduce();
  sw.warp_reduce();
  // CTA-level reduction first: one atomic per statistic per CTA (same-line
  // atomics from every warp of every CTA queued up in front of the barrier)
  __shared__ float red[kConsumers / 32][4];
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5][0] = sx.amax;
    red[threadIdx.x >> 5][1] = sx.mnz;
    red[threadIdx.x >> 5][2] = sw.amax;
    red[threadIdx.x >> 5][3] = sw.mnz;
  }
  asm volatile("bar.sync 2, %0;" ::"n"(kConsumers) : "memory");
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < kConsumers / 32; ++w) {
      asm("max.NaN.f32 %0, %0, %1;" : "+f"(sx.amax) : "f"(red[w][0]));
      asm("min.f32 %0, %0, %1;" : "+f"(sx.mnz) : "f"(red[w][1]));
      asm("max.NaN.f32 %0, %0, %1;" : "+f"(sw.amax) : "f"(red[w][2]));
      asm("min.f32 %0, %0, %1;" : "+f"(sw.mnz) : "f"(red[w][3]));
    }
    if (GX) sx.commit(a.stats);
    if (GW) sw.commit(a.stats + 2);
  }
  if (MODE == kStats) return;
  // ---------------- grid barrier (consumer threads only; all CTAs co-resident)
  grid_barrier(a.stats + 32, gridDim.x, a.poll_ns);
  stamp(2);
  consume_quant<T, GX, GW, BM, kDyn, GRP>(a, tiles, full, empty, meta, cbuf, slot, phase, true);
  stamp(3);
  if (GW && a.cs_out) {
    // column sums: one warp per column, lanes over the column's contiguous
    // row-group partials (coalesced, 16 loads in flight per lane), fixed
    // summation order and shuffle tree -> deterministic.  The partials were
    // written before the grid barrier (L2 loads).
    if (a.dev_flags & 4) {  // partials written by the QUANT pass
      asm volatile("bar.sync 2, %0;" ::"n"(kConsumers) : "memory");
      grid_barrier(a.stats + 32, 2 * gridDim.x, a.poll_ns);
    }
    const int lane = threadIdx.x & 31;
    for (int c = blockIdx.x * (kConsumers / 32) + (threadIdx.x >> 5); c < a.cols;
         c += gridDim.x * (kConsumers / 32)) {
      const float* p = a.cs_part + int64_t(c) * a.groups;
      float acc = 0.0f;
      for (int g0 = 0; g0 < a.groups; g0 += 16 * 32) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int g = g0 + 32 * j + lane;
          v[j] = g < a.groups ? __ldcg(p + g) : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) a.cs_out[c] = acc;
    }
  }
  stamp(4);
  // this CTA's outputs are written: a dependent GEMM launched with programmatic
  // serialization may start its prologue (it waits for the whole grid before reading)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (MODE == kBoth && a.self_reset) {
    // library-owned statistics slot: the last CTA to get here (every other CTA
    // is past both passes and every barrier) zeroes it for its next launch
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.stats + 33) : "memory");
      if (old == gridDim.x - 1) {
        for (int i = 0; i < HLQ_STATS_WS_BYTES / 4; ++i)
          asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(a.stats + i), "r"(0u) : "memory");
      }
    }
  }
}

template <typename T, int MODE, bool GX, bool GW, int BM, int GRP>
void launch_one(const CUtensorMap& map, Args a, cudaStream_t stream) {
  constexpr int kRow = Tr<T>::kRow;
  const size_t smem = 128 + size_t(kStages) * 16 * kRow +
                      (GW && MODE != kStats ? size_t(a.cbw) * a.cstride : 0) + 8 + 2 * kStages * 8 + kStages * kMetaWords * 4 + 8;
  auto kern = tma_tile_kernel<T, MODE, GX, GW, BM, GRP>;
  static std::atomic<unsigned long long> attr{0};  // per template instance and device
  smem_attr_once(reinterpret_cast<const void*>(kern), 200 * 1024, attr);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  if (per_sm > HLQ_TR_MINB) per_sm = HLQ_TR_MINB;  // 5 resident CTAs measured no faster (more tail per item)
  static const int knob_cps = env_knob("HLQ_TR_CTAS_PER_SM");  // development sweeps
  if (knob_cps >= 1 && knob_cps < per_sm) per_sm = knob_cps;

  const int cap = num_sms() * per_sm;
  const int grid = a.items < 1 ? 1 : (a.items > cap ? cap : a.items);
  if (MODE != kBoth) {
    kern<<<grid, kThreads, smem, stream>>>(map, a);
    return;
  }
  // every CTA must be resident for the grid barrier: cooperative launch
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr_coop[2];
  attr_coop[0].id = cudaLaunchAttributeCooperative;
  attr_coop[0].val.cooperative = 1;
  // programmatic dependent launch (the kernel waits on griddepcontrol before its
  // first read); HLQ_PDL=0 or a runtime that rejects the combination: plain
  static const int pdl_off = env_knob("HLQ_PDL");
  attr_coop[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_coop[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_coop;
  cfg.numAttrs = pdl_off == 0 ? 1 : 2;
  if (cudaLaunchKernelEx(&cfg, kern, map, a) != cudaSuccess && cfg.numAttrs == 2) {
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, map, a);
  }
}

template <typename T, int MODE, bool GX, bool GW>
void launch_bm(const CUtensorMap& map, const Args& a, cudaStream_t st) {
  if (a.tq > 1) {  // grouped narrow tiles: the default plan or the generic bitmap
    const bool conv = a.taps != 0;
    if (GW && a.bitmap == 0x5555) {
      if (conv) return launch_one<T, MODE, GX, GW, 0x5555, 1>(map, a, st);
      return launch_one<T, MODE, GX, GW, 0x5555, 2>(map, a, st);
    }
    if (conv) return launch_one<T, MODE, GX, GW, 0, 1>(map, a, st);
    return launch_one<T, MODE, GX, GW, 0, 2>(map, a, st);
  }
  if (!GW) return launch_one<T, MODE, GX, GW, 0, 0>(map, a, st);
  switch (a.bitmap) {
    case 0x5555: return launch_one<T, MODE, GX, GW, 0x5555, 0>(map, a, st);  // rank 8 (default plan)
    case 0x1111: return launch_one<T, MODE, GX, GW, 0x1111, 0>(map, a, st);  // rank 4
    case 0x0101: return launch_one<T, MODE, GX, GW, 0x0101, 0>(map, a, st);  // rank 2
    case 0xFFFF: return launch_one<T, MODE, GX, GW, 0xFFFF, 0>(map, a, st);  // full (H.W, rank 16)
    default: return launch_one<T, MODE, GX, GW, 0, 0>(map, a, st);           // calibrated bases
  }
}

template <typename T, int MODE>
void launch_ops(const CUtensorMap& map, const Args& a, bool gx, bool gw, cudaStream_t st) {
  if (gx && gw) launch_bm<T, MODE, true, true>(map, a, st);
  else if (gx) launch_bm<T, MODE, true, false>(map, a, st);
  else launch_bm<T, MODE, false, true>(map, a, st);
}

template <typename T>
void launch_modes(const CUtensorMap& map, const Args& a, int mode, bool gx, bool gw, cudaStream_t st) {
  if (mode == kStats) launch_ops<T, kStats>(map, a, gx, gw, st);
  else if (mode == kQuant) launch_ops<T, kQuant>(map, a, gx, gw, st);
  else launch_ops<T, kBoth>(map, a, gx, gw, st);
}

int tr_poll_ns() {
  static const int f = env_knob("HLQ_TR_POLL_NS");
  return f > 0 ? f : 128;
}

int tr_dev_flags() {
  static const int f = env_knob("HLQ_TR_FLAGS");
  return f > 0 ? f : 0;
}

// Blocks per work item: >= 32-byte output runs per column when the problem is
// large, while keeping >= ~3 work items per SM.
int choose_nb(int total_blocks, int cols, int rank) {
  int nb = rank >= 8 ? 4 : (rank >= 4 ? 8 : 16);
  const int ncol_tiles = (cols + kCols - 1) / kCols;
  while (nb > 1 && ((total_blocks + nb - 1) / nb) * ncol_tiles < num_sms() * 3) nb >>= 1;
  static const int knob_nb = env_knob("HLQ_TR_NB");  // development sweeps
  if (knob_nb >= 1 && knob_nb <= 16) nb = knob_nb;
  return nb;
}

// Column sums without the fused path (sources the tensor map cannot describe):
// one thread per column over every row, in row order (deterministic).
template <typename T>
__global__ void colsum_kernel(const T* src, int64_t segs, int64_t rows, int64_t cols, int64_t ld, int64_t seg,
                              float* out) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float acc = 0.0f;
  for (int64_t s = 0; s < segs; ++s)
    for (int64_t r = 0; r < rows; ++r) {
      const T v = src[s * seg + r * ld + c];
      acc += sizeof(T) == 2 ? __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(&v))
                            : *reinterpret_cast<const float*>(&v);
    }
  out[c] = acc;
}

void launch_colsum(const TransformArgs& t, cudaStream_t st) {
  const int grid = int((t.cols + 127) / 128);
  if (t.dtype == kBF16)
    colsum_kernel<<<grid, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(t.src), t.segs, t.rows, t.cols,
                                        t.ld_src, t.seg_src, t.colsum_out);
  else
    colsum_kernel<<<grid, 128, 0, st>>>(static_cast<const float*>(t.src), t.segs, t.rows, t.cols, t.ld_src,
                                        t.seg_src, t.colsum_out);
}

}  // namespace

__device__ uint32_t g_nonfinite_flag;
__device__ uint32_t g_stat_slots[kStatSlots][HLQ_STATS_WS_BYTES / 4];  // zero-initialised

uint32_t* stats_slot() {
  static uint32_t* base[64] = {nullptr};
  static std::atomic<uint32_t> next[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!base[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_stat_slots) != cudaSuccess) return nullptr;
    base[dev] = static_cast<uint32_t*>(p);
  }
  const uint32_t i = next[dev].fetch_add(1u, std::memory_order_relaxed) % kStatSlots;
  return base[dev] + size_t(i) * (HLQ_STATS_WS_BYTES / 4);
}

uint32_t* nonfinite_word() {
  static uint32_t* addr[64] = {nullptr};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!addr[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_nonfinite_flag) != cudaSuccess) return nullptr;
    addr[dev] = static_cast<uint32_t*>(p);
  }
  return addr[dev];
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool launch_conv_acbp_tma(const void* x, int dtype, int B, int H, int W, int C, int k, int stride, int pad,
                          uint32_t bitmap, int bits, int mode, uint32_t* stats, int8_t* dst, int64_t ld_dst,
                          float* scale, cudaStream_t stream, bool pooled) {
  static EncodeIm2colFn enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeIm2colFn>(p);
    return EncodeIm2colFn(nullptr);
  }();
  const size_t esz = dtype == kBF16 ? 2 : 4;
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (!enc || (reinterpret_cast<uintptr_t>(x) % 16) || (size_t(C) * esz) % 16 || stride > 8 || pad > 127 ||
      k - 1 - pad > 127 || k > 16 || Ho * Wo < 16)
    return false;
  // narrow inputs: several taps per 256-column step, one C-channel im2col box each
  static const bool nogroup_conv = env_knob("HLQ_CONV_NOGROUP") != -1;
  const int tq = (C == 32 || C == 64 || C == 128) && !nogroup_conv ? kCols / C : 1;
  CUtensorMap map;
  const cuuint64_t dims[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(B)};
  const cuuint64_t strides[3] = {cuuint64_t(C) * esz, cuuint64_t(C) * esz * W, cuuint64_t(C) * esz * W * H};
  const int lower[2] = {-pad, -pad};
  const int upper[2] = {pad - (k - 1), pad - (k - 1)};
  const cuuint32_t es[4] = {1, cuuint32_t(stride), cuuint32_t(stride), 1};
  if (enc(&map, dtype == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
          const_cast<void*>(x), dims, strides, lower, upper, cuuint32_t(tq > 1 ? C : kCols), 16, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  Args a{};
  a.rows = Ho * Wo;
  a.cols = C;
  a.nblk = (a.rows + 15) / 16;
  a.total_blocks = B * a.nblk;
  a.rank = __builtin_popcount(bitmap);
  a.taps = k * k;
  a.kconv = k;
  a.cstr = stride;
  a.cpad = pad;
  a.wo_n = Wo;
  a.ncol_tiles = (C + kCols - 1) / kCols;
  a.tq = tq;
  a.cch = C;
  a.vblocks = a.total_blocks;
  a.cbw = kCols;
  // row sharing (see Args): only the middle tap row is transformed
  static const bool noshare = env_knob("HLQ_CONV_NOSHARE") == 1;
  const bool share = !noshare && stride == 1 && (k & 1) && pad == (k - 1) / 2 && k > 1 && Ho == H &&
                     Wo % 16 == 0 && a.rank == 8;
  a.tap0 = share ? pad * k : 0;
  a.ntap_c = share ? k : a.taps;
  a.sh_blk = Wo / 16;
  const int ntg = (a.ntap_c + tq - 1) / tq;  // tap groups per (pixel block, column tile)
  {
    int nb = a.rank >= 8 ? 4 : (a.rank >= 4 ? 8 : 16);
    while (nb > 1 && ((a.total_blocks + nb - 1) / nb) * a.ncol_tiles * ntg < num_sms() * 3) nb >>= 1;
    a.nb = nb;
  }
  // the flush addresses whole items inside one image (blocks per image a multiple of nb)
  a.share = share && a.nblk % a.nb == 0 ? 1 : 0;
  if (share && !a.share) {
    a.tap0 = 0;
    a.ntap_c = a.taps;
  }
  a.items = ((a.total_blocks + a.nb - 1) / a.nb) * a.ncol_tiles * ((a.ntap_c + tq - 1) / tq);
  a.bitmap = bitmap;
  a.bits_gx = bits;
  a.bits_gw = bits;
  a.stats = stats;
  a.dst_gw = dst;
  a.ld_gw = ld_dst;
  a.scale_gw = scale;
  a.nonfinite = nonfinite_word();
  a.cstride = a.nb * a.rank + 16;
  a.self_reset = pooled && mode == kBoth ? 1 : 0;
  a.dev_flags = tr_dev_flags();
  a.poll_ns = tr_poll_ns();
  if (dtype == kBF16)
    launch_modes<__nv_bfloat16>(map, a, mode, false, true, stream);
  else
    launch_modes<float>(map, a, mode, false, true, stream);
  return true;
}

#ifdef HLQ_TR_TRACE
unsigned long long* g_tr_trace = nullptr;
#endif

void launch_transform(const TransformArgs& t, int mode, cudaStream_t stream) {
  const size_t esz = t.dtype == kBF16 ? 2 : 4;
  const bool fits32 = t.rows < (int64_t(1) << 30) && t.cols < (int64_t(1) << 30) &&
                      t.segs * ((t.rows + 15) / 16) < (int64_t(1) << 30);
  const bool aligned = (reinterpret_cast<uintptr_t>(t.src) % 16 == 0) && ((t.ld_src * esz) % 16 == 0) &&
                       (t.segs <= 1 || (t.seg_src * esz) % 16 == 0);
  CUtensorMap map;
  bool ok = fits32 && aligned && t.rows > 0 && t.cols > 0 && t.segs > 0;
  // narrow sources: row groups of 256 / cols blocks per step (one cols-wide box each)
  static const bool nogroup = env_knob("HLQ_TR_NOGROUP") != -1;
  const int tq = (t.cols == 32 || t.cols == 64 || t.cols == 128) && !nogroup
                     ? int(kCols / t.cols) : 1;
  if (ok) {
    const uint64_t seg_stride = t.segs > 1 ? uint64_t(t.seg_src) * esz
                                           : (uint64_t(t.rows) * t.ld_src * esz + 15) & ~uint64_t(15);
    const uint64_t dims[3] = {uint64_t(t.cols), uint64_t(t.rows), uint64_t(t.segs)};
    const uint64_t strides[2] = {uint64_t(t.ld_src) * esz, seg_stride};
    const uint32_t box[3] = {uint32_t(tq > 1 ? t.cols : kCols), 16, 1};
    ok = encode_tensor_map(&map, t.dtype == kBF16 ? 1 : 2, 3, t.src, dims, strides, box, 0);
  }
  if (!ok) {
    if (t.pooled) cudaMemsetAsync(t.stats, 0, HLQ_STATS_WS_BYTES, stream);  // not self-cleaning
    if (mode == kBoth) {
      launch_transform_fallback(t, kStats, stream);
      launch_transform_fallback(t, kQuant, stream);
    } else {
      launch_transform_fallback(t, mode, stream);
    }
    if (t.colsum_out) launch_colsum(t, stream);
    // the fallback kernels do not clean up after themselves: leave the slot zeroed
    if (t.pooled) cudaMemsetAsync(t.stats, 0, HLQ_STATS_WS_BYTES, stream);
    return;
  }
  Args a{};
  a.rows = int(t.rows);
  a.cols = int(t.cols);
  a.nblk = int((t.rows + 15) / 16);
  a.total_blocks = int(t.segs) * a.nblk;
  a.rank = t.do_gw ? __builtin_popcount(t.bitmap) : 0;
  a.tq = tq;
  a.cch = tq > 1 ? a.cols : kCols;
  a.vblocks = (a.total_blocks + tq - 1) / tq;
  a.cbw = tq > 1 ? a.cols : kCols;
  a.nb = t.do_gw ? choose_nb(a.vblocks, tq > 1 ? kCols : a.cols, a.rank * tq) : 4;
  a.ncol_tiles = (a.cols + kCols - 1) / kCols;
  a.items = ((a.vblocks + a.nb - 1) / a.nb) * a.ncol_tiles;
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
  a.nonfinite = nonfinite_word();
  a.pack_gx = t.pack_gx ? 1 : 0;
  a.cstride = a.nb * a.tq * a.rank + 16;
  a.dev_flags = tr_dev_flags();
  a.poll_ns = tr_poll_ns();
  a.self_reset = t.pooled && mode == kBoth ? 1 : 0;
  {
    // keep ~HLQ_TR_KEEP_MB (default 32) MB of the source resident between the passes
    // (fc2-input ACBP 75.8 -> 71.7 us, fc1 gy dual 120.7 -> 118.8 us; 64 / 96 MB no better)
    static const int knob_keep = env_knob("HLQ_TR_KEEP_MB");
    const double keep_mb = knob_keep >= 0 ? double(knob_keep) : 32.0;
    const double src_mb = double(t.segs) * double(t.rows) * double(t.cols) * double(esz) / 1048576.0;
    a.keep_items = keep_mb <= 0.0 ? 0 : (src_mb <= keep_mb ? a.items : int(double(a.items) * keep_mb / src_mb));
  }
  if (t.pooled && mode != kBoth) cudaMemsetAsync(t.stats, 0, HLQ_STATS_WS_BYTES, stream);
#ifdef HLQ_TR_TRACE
  a.trace = g_tr_trace;
#endif
  if (t.colsum_out && mode == kBoth && t.do_gw) {
    a.groups = ((a.vblocks + a.nb - 1) / a.nb) * a.tq;  // rg: one partial per sub-tile position
    a.cs_part = t.colsum_ws;
    a.cs_out = t.colsum_out;
  }
  if (t.dtype == kBF16)
    launch_modes<__nv_bfloat16>(map, a, mode, t.do_gx, t.do_gw, stream);
  else
    launch_modes<float>(map, a, mode, t.do_gx, t.do_gw, stream);
  if (t.colsum_out && !a.cs_out) launch_colsum(t, stream);
  if (t.pooled && mode != kBoth) cudaMemsetAsync(t.stats, 0, HLQ_STATS_WS_BYTES, stream);  // leave it zeroed
}

size_t transform_colsum_ws(int64_t segs, int64_t rows, int64_t cols, uint32_t bitmap) {
  if (segs <= 0 || rows <= 0 || cols <= 0) return 0;
  const int64_t total_blocks = segs * ((rows + 15) / 16);
  if (total_blocks >= (int64_t(1) << 30) || cols >= (int64_t(1) << 30)) return 0;
  (void)bitmap;  // upper bound over the item sizes and row groups the launch may choose
  return size_t(total_blocks + 16 * 16) * size_t(cols) * sizeof(float);
}

}  // namespace hlq

#ifdef HLQ_TR_TRACE
extern "C" __attribute__((visibility("default"))) void hlq_debug_set_trace(unsigned long long* p) {
  hlq::g_tr_trace = p;
}
#endif
