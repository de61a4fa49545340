// Batched W codes: Q_b(HT_O(W)) for many weight matrices in ONE cooperative
// launch (hq_grad_input's right operand, backprop.py:363,368, per layer).
//
// In training every weight changes at each optimizer step, so the dX operand
// of every HLQ layer needs fresh codes once per step.  Per layer that is a
// small tensor (0.6-9.4 MB fp32 in ViT-B/16) whose two-pass transform is
// dominated by fixed costs (launch, first loads, the grid-wide scale
// dependency); doing all 49 layers of the model in one launch amortises them.
//
// W is (O, I) fp32 row-major; the transform runs along O (blocks of 16 rows,
// zero rows past O), codes are written K-major as (I, ld >= pad16(O)) -- the
// same layout, values and per-tensor scale as hlq_quantize_proj_rows(W, 1, O,
// I, bitmap 0xFFFF) (bit-identical: same butterfly, statistics and quantizer).
//
// Work item = (tensor, 16-row block, 256-column chunk); a 128-thread CTA runs
// one item at a time, thread t owning columns (2t, 2t+1): 16 coalesced 8-byte
// loads, the 16-point butterfly on f32x2 lanes, then statistics (pass 1) or
// codes (pass 2, two 16-byte stores).  Pass 1 -> per-tensor atomic max ->
// grid barrier -> pass 2.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "hlq_internal.h"
#include "hlq_quant.cuh"

namespace hlq {

namespace {

using namespace dev;

constexpr int kThr = 128;
constexpr int kColsPerItem = 2 * kThr;

struct WDesc {
  const float* w;
  __nv_bfloat16* wbf;  // optional bf16 copy of W (the forward GEMM's operand under autocast)
  int8_t* codes;
  float* scale;
  uint32_t* stats;  // 8 words per tensor: {amax, ~minnz, ...}
  int64_t ld;
  int O, I, nblk, nchunk, item0;
};

struct WBatch {
  WDesc t[kMaxWeights];
  int n, items, bits;
  uint32_t* barrier;
  uint32_t* nonfinite;  // nonfinite_word()
};

__device__ __forceinline__ int find_tensor(const WBatch& b, int item) {
  int lo = 0, hi = b.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b.t[mid].item0 <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <bool FAST>
__device__ __forceinline__ void quant_item(const WDesc& d, int blk, int c0, const Quant& q) {
  const int c = c0 + 2 * int(threadIdx.x);
  if (c >= d.I) return;
  float2 p[16];
  const bool two = c + 1 < d.I;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int o = blk * 16 + r;
    p[r] = make_float2(0.0f, 0.0f);
    if (o < d.O) {
      const float* src = d.w + int64_t(o) * d.I + c;
      if (two && (reinterpret_cast<uintptr_t>(src) & 7) == 0) p[r] = __ldg(reinterpret_cast<const float2*>(src));
      else { p[r].x = __ldg(src); if (two) p[r].y = __ldg(src + 1); }
    }
  }
  fwht16_pair(p);
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = quant2<FAST>(p[i], q);  // (code col c, code col c+1)
  uint32_t cx[4], cy[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t t01 = __byte_perm(w[4 * k], w[4 * k + 1], 0x6420);
    const uint32_t t23 = __byte_perm(w[4 * k + 2], w[4 * k + 3], 0x6420);
    cx[k] = __byte_perm(t01, t23, 0x6420);
    cy[k] = __byte_perm(t01, t23, 0x7531);
  }
  *reinterpret_cast<uint4*>(d.codes + int64_t(c) * d.ld + blk * 16) = make_uint4(cx[0], cx[1], cx[2], cx[3]);
  if (two)
    *reinterpret_cast<uint4*>(d.codes + int64_t(c + 1) * d.ld + blk * 16) = make_uint4(cy[0], cy[1], cy[2], cy[3]);
}

__global__ void __launch_bounds__(kThr) weight_codes_kernel(const __grid_constant__ WBatch b) {
  // ---------------- pass 1: statistics
  for (int item = blockIdx.x; item < b.items; item += gridDim.x) {
    const int ti = find_tensor(b, item);
    const WDesc& d = b.t[ti];
    const int local = item - d.item0;
    const int blk = local / d.nchunk, c0 = (local - blk * d.nchunk) * kColsPerItem;
    const int c = c0 + 2 * int(threadIdx.x);
    Stat st;
    if (c < d.I) {
      float2 p[16];
      const bool two = c + 1 < d.I;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int o = blk * 16 + r;
        p[r] = make_float2(0.0f, 0.0f);
        if (o < d.O) {
          const float* src = d.w + int64_t(o) * d.I + c;
          if (two && (reinterpret_cast<uintptr_t>(src) & 7) == 0) p[r] = __ldg(reinterpret_cast<const float2*>(src));
          else { p[r].x = __ldg(src); if (two) p[r].y = __ldg(src + 1); }
          if (d.wbf) {  // the bf16 cast of W rides on the statistics pass's read
            __nv_bfloat16* dst = d.wbf + int64_t(o) * d.I + c;
            if (two && (reinterpret_cast<uintptr_t>(dst) & 3) == 0)
              *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(p[r].x, p[r].y);
            else { dst[0] = __float2bfloat16_rn(p[r].x); if (two) dst[1] = __float2bfloat16_rn(p[r].y); }
          }
        }
      }
      fwht16_pair(p);
#pragma unroll
      for (int i = 0; i < 16; ++i) st.add2(p[i].x, p[i].y);
    }
    st.warp_reduce();
    if ((threadIdx.x & 31) == 0) st.commit(d.stats);
  }
  // ---------------- grid barrier (all CTAs co-resident: cooperative launch)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(b.barrier, 1u);
    uint32_t seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(b.barrier) : "memory");
      if (seen < gridDim.x) __nanosleep(64);
    } while (seen < gridDim.x);
  }
  __syncthreads();
  // ---------------- pass 2: codes (reverse order: the last items are in L2)
  int cur = -1;
  Quant q{};
  for (int k = blockIdx.x; k < b.items; k += gridDim.x) {
    const int item = b.items - 1 - k;
    const int ti = find_tensor(b, item);
    const WDesc& d = b.t[ti];
    if (ti != cur) {
      q = make_quant(d.stats, b.bits);
      cur = ti;
      if (item == d.item0 && threadIdx.x == 0 && d.scale) *d.scale = q.s;
      if (item == d.item0 && threadIdx.x == 0) flag_nonfinite(q, b.nonfinite);
    }
    const int local = item - d.item0;
    const int blk = local / d.nchunk, c0 = (local - blk * d.nchunk) * kColsPerItem;
    if (q.fast) quant_item<true>(d, blk, c0, q);
    else quant_item<false>(d, blk, c0, q);
  }
}

}  // namespace

int launch_weight_codes(int n, const float* const* w, const int64_t* O, const int64_t* I, int bits,
                        int8_t* const* codes, const int64_t* ld, float* const* scales, uint32_t* ws,
                        cudaStream_t stream, void* const* wbf16) {
  WBatch b{};
  b.n = n;
  b.bits = bits;
  int items = 0;
  for (int i = 0; i < n; ++i) {
    WDesc& d = b.t[i];
    d.w = w[i];
    d.wbf = wbf16 ? static_cast<__nv_bfloat16*>(wbf16[i]) : nullptr;
    d.codes = codes[i];
    d.scale = scales[i];
    d.stats = ws + 8 * i;
    d.ld = ld[i];
    d.O = int(O[i]);
    d.I = int(I[i]);
    d.nblk = (d.O + 15) / 16;
    d.nchunk = (d.I + kColsPerItem - 1) / kColsPerItem;
    d.item0 = items;
    items += d.nblk * d.nchunk;
  }
  b.items = items;
  b.barrier = ws + 8 * n;
  b.nonfinite = nonfinite_word();
  cudaError_t e = cudaMemsetAsync(ws, 0, size_t(8 * n + 8) * sizeof(uint32_t), stream);
  if (e != cudaSuccess) return int(e);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, weight_codes_kernel, kThr, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int cap = num_sms() * per_sm;
  const int grid = items < cap ? items : cap;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThr);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return int(cudaLaunchKernelEx(&cfg, weight_codes_kernel, b));
}

}  // namespace hlq
