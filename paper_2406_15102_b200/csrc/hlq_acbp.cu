// ACBP container on the GPU (reference acbp.py:3-212): the
// bit-exact serialized form of the compressed activation -- header, per-tensor
// scale, payload in the reference's C order (int8 raw, or int4 packed two per
// byte, low nibble first) and a zlib CRC32 of every prior byte.
//
//   pack:   payload transpose (our K-major (R, K) codes -> reference (K, R)
//           order: element e = k*R + r) + nibble packing, header bytes written
//           on the device (the scale never leaves it), then CRC32.
//   unpack: header parsed on the host (33 bytes copied back; every field
//           validated with the reference's messages and byte offsets), then
//           on the device: payload range check (first bad byte via atomicMin),
//           padding-nibble check, CRC32, transpose back to K-major.
//
// CRC32 (reflected 0xEDB88320, init/xor 0xFFFFFFFF) in parallel: the register
// update is linear, update(s, D) = shift(s, |D|) ^ update(0, D), where
// shift(s, n) = s run through n zero bytes (a GF(2)-linear map, applied with
// four 256-entry tables per power-of-two length).  The message is treated as
// right-aligned in a power-of-two number of 16 KiB chunks (leading zeros keep a
// zero-state CRC at zero), so every combine is between equal power-of-two
// blocks: a thread reduces 64 bytes with slicing-by-16 tables, a warp shuffle
// tree and a CTA tree combine a chunk (persistent CTAs; all-padding chunks are
// skipped), one 1024-thread CTA folds the chunk CRCs, and the 0xFFFFFFFF
// initial register enters as shift(0xFFFFFFFF, n).  The payload transposes
// move warp-wide runs of 32 consecutive bytes through a shared tile (the
// payload starts at the unaligned byte 33).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "hlq_internal.h"

namespace hlq {

namespace {

constexpr int kPow = 40;  // shift tables for 2^j bytes, j = 0..39

__device__ uint32_t g_crc_tab[256];
__device__ uint32_t g_crc_pow[kPow][4][256];
__device__ uint32_t g_crc_s16[16][256];  // slicing-by-16 tables (crc16_step)

uint32_t host_tab[256];

// shift(x, 2^j bytes) as 4 byte-sliced tables; level j+1 = level j applied twice
void host_tables(uint32_t (*pw)[4][256]) {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
    host_tab[i] = c;
  }
  for (int b = 0; b < 4; ++b)
    for (uint32_t v = 0; v < 256; ++v) {
      const uint32_t r = v << (8 * b);
      pw[0][b][v] = host_tab[r & 0xFFu] ^ (r >> 8);  // one zero byte
    }
  for (int j = 1; j < kPow; ++j)
    for (int b = 0; b < 4; ++b)
      for (uint32_t v = 0; v < 256; ++v) {
        uint32_t r = v << (8 * b);
        for (int t = 0; t < 2; ++t)
          r = pw[j - 1][0][r & 0xFFu] ^ pw[j - 1][1][(r >> 8) & 0xFFu] ^ pw[j - 1][2][(r >> 16) & 0xFFu] ^
              pw[j - 1][3][r >> 24];
        pw[j][b][v] = r;
      }
}

// Upload the tables once per device (static module memory; no allocation).
bool ensure_tables() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return false;
  std::lock_guard<std::mutex> lock(mu);
  if (done[dev]) return true;
  static uint32_t pw[kPow][4][256];
  static bool built = false;
  if (!built) {
    host_tables(pw);
    built = true;
  }
  static uint32_t s16[16][256];
  for (uint32_t v = 0; v < 256; ++v) s16[0][v] = host_tab[v];
  for (int k = 1; k < 16; ++k)
    for (uint32_t v = 0; v < 256; ++v) s16[k][v] = (s16[k - 1][v] >> 8) ^ host_tab[s16[k - 1][v] & 0xFFu];
  if (cudaMemcpyToSymbol(g_crc_tab, host_tab, sizeof(host_tab)) != cudaSuccess) return false;
  if (cudaMemcpyToSymbol(g_crc_s16, s16, sizeof(s16)) != cudaSuccess) return false;
  if (cudaMemcpyToSymbol(g_crc_pow, pw, sizeof(pw)) != cudaSuccess) return false;
  done[dev] = true;
  return true;
}

__device__ __forceinline__ uint32_t shift_pow(uint32_t x, int j) {
  return __ldg(&g_crc_pow[j][0][x & 0xFFu]) ^ __ldg(&g_crc_pow[j][1][(x >> 8) & 0xFFu]) ^
         __ldg(&g_crc_pow[j][2][(x >> 16) & 0xFFu]) ^ __ldg(&g_crc_pow[j][3][x >> 24]);
}

// Slicing-by-16 tables: T_k[v] = the register after byte v and k zero bytes
// (T_0 = the byte table); a 16-byte block b0..b15 updates a register c as
// c' = T15[(c ^ w0) & 0xFF] ^ T14[(c ^ w0) >> 8 & 0xFF] ^ ... ^ T0[b15].
__device__ __forceinline__ uint32_t crc16_step(uint32_t c, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
  const uint32_t x = c ^ w0;
  const uint32_t(*t)[256] = g_crc_s16;
  return __ldg(&t[15][x & 0xFFu]) ^ __ldg(&t[14][(x >> 8) & 0xFFu]) ^ __ldg(&t[13][(x >> 16) & 0xFFu]) ^
         __ldg(&t[12][x >> 24]) ^ __ldg(&t[11][w1 & 0xFFu]) ^ __ldg(&t[10][(w1 >> 8) & 0xFFu]) ^
         __ldg(&t[9][(w1 >> 16) & 0xFFu]) ^ __ldg(&t[8][w1 >> 24]) ^ __ldg(&t[7][w2 & 0xFFu]) ^
         __ldg(&t[6][(w2 >> 8) & 0xFFu]) ^ __ldg(&t[5][(w2 >> 16) & 0xFFu]) ^ __ldg(&t[4][w2 >> 24]) ^
         __ldg(&t[3][w3 & 0xFFu]) ^ __ldg(&t[2][(w3 >> 8) & 0xFFu]) ^ __ldg(&t[1][(w3 >> 16) & 0xFFu]) ^
         __ldg(&t[0][w3 >> 24]);
}

// The message is right-aligned in a virtual buffer of nch (a power of two)
// chunks of 16 KiB: leading zero bytes leave a zero-state CRC at zero, so every
// chunk is full and every combine below is between equal power-of-two blocks.
// A thread reduces 64 bytes (4 slicing-by-16 steps), a warp shuffle tree and
// a CTA tree combine them (shift by 2^j bytes = 4 byte-sliced table lookups);
// chunks that lie wholly in the virtual padding are zero and skipped.
constexpr int kPiece16 = 64;
constexpr int kChunk16 = 256 * kPiece16;  // 16 KiB per CTA iteration

__global__ void __launch_bounds__(256) crc_chunks16_kernel(const uint8_t* __restrict__ buf, int64_t n, int64_t vpad,
                                                           int64_t nch, bool aligned, uint32_t* __restrict__ out) {
  __shared__ uint32_t part[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const int64_t c0 = ch * kChunk16 - vpad;  // real offset of the chunk's first byte
    if (c0 + kChunk16 <= 0) {                 // all virtual zeros
      if (threadIdx.x == 0) out[ch] = 0;
      continue;
    }
    const int64_t o = c0 + int64_t(threadIdx.x) * kPiece16;
    uint32_t w[16];
    if (aligned && o >= 0 && o + kPiece16 <= n && (o & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(buf + o) + q);
        w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
      }
    } else if (aligned && o >= 4 && o + kPiece16 + 4 <= n) {
      // the chunk grid is offset from the buffer by the (uniform) virtual
      // padding: 17 aligned words, funnel-shifted by the byte misalignment
      const uint32_t* base = reinterpret_cast<const uint32_t*>(buf + (o & ~int64_t(3)));
      const uint32_t sh = 8u * uint32_t(o & 3);
      uint32_t W[17];
#pragma unroll
      for (int q = 0; q < 17; ++q) W[q] = __ldg(base + q);
#pragma unroll
      for (int q = 0; q < 16; ++q) w[q] = __funnelshift_r(W[q], W[q + 1], sh);
    } else {  // unaligned or at the message edges: bytes (zero outside [0, n))
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        uint32_t x = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int64_t a = o + 4 * q + b;
          if (a >= 0 && a < n) x |= uint32_t(__ldg(buf + a)) << (8 * b);
        }
        w[q] = x;
      }
    }
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) c = crc16_step(c, w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
#pragma unroll
    for (int j = 0; j < 5; ++j) {  // blocks of 64 << j bytes
      const uint32_t later = __shfl_down_sync(0xffffffffu, c, 1 << j);
      if ((lane & ((2 << j) - 1)) == 0) c = shift_pow(c, 6 + j) ^ later;
    }
    if (lane == 0) part[warp] = c;
    __syncthreads();
    if (warp == 0) {
      c = lane < 8 ? part[lane] : 0u;
#pragma unroll
      for (int j = 0; j < 3; ++j) {  // blocks of 2 KiB << j
        const uint32_t later = __shfl_down_sync(0xffffffffu, c, 1 << j);
        if ((lane & ((2 << j) - 1)) == 0) c = shift_pow(c, 11 + j) ^ later;
      }
      if (lane == 0) out[ch] = c;
    }
    __syncthreads();
  }
}

// one CTA: each thread folds nch/1024 consecutive chunk CRCs, then a warp
// shuffle tree and a CTA tree over equal blocks; zlib crc32 = raw ^
// shift(0xFFFFFFFF, n) ^ 0xFFFFFFFF.  The stored CRC (the container's last 4
// bytes, when `stored` is given) is copied next to the computed one so the
// host reads both with one copy.
__global__ void __launch_bounds__(1024) crc_finish16_kernel(const uint32_t* __restrict__ chunks, int64_t nch, int64_t n,
                                                            uint8_t* dst, uint32_t* value_out,
                                                            const uint8_t* stored) {
  __shared__ uint32_t part[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = nch >= 1024 ? nch / 1024 : 1;
  const int active = int(nch >= 1024 ? 1024 : nch);
  uint32_t r = 0;
  if (int(threadIdx.x) < active)
    for (int64_t c = threadIdx.x * per; c < (threadIdx.x + 1) * per; ++c) r = shift_pow(r, 14) ^ chunks[c];
  int lg = 14;  // log2 bytes of one thread's block
  for (int64_t p = per; p > 1; p >>= 1) ++lg;
  // the tree spans the first `active` (a power of two) entries only: entries
  // past the message would act as trailing zero bytes
  int levels = 0;
  while ((1 << levels) < active) ++levels;
  for (int j = 0; j < 5 && j < levels; ++j) {
    const uint32_t later = __shfl_down_sync(0xffffffffu, r, 1 << j);
    if ((lane & ((2 << j) - 1)) == 0) r = shift_pow(r, lg + j) ^ later;
  }
  if (lane == 0) part[warp] = r;
  __syncthreads();
  if (warp == 0) {
    r = part[lane];
    for (int j = 0; j + 5 < levels; ++j) {
      const uint32_t later = __shfl_down_sync(0xffffffffu, r, 1 << j);
      if ((lane & ((2 << j) - 1)) == 0) r = shift_pow(r, lg + 5 + j) ^ later;
    }
    if (lane == 0) {
      uint32_t init = 0xFFFFFFFFu;
      for (int j = 0; j < kPow; ++j)
        if ((n >> j) & 1) init = shift_pow(init, j);
      const uint32_t crc = r ^ init ^ 0xFFFFFFFFu;
      if (dst)
        for (int b = 0; b < 4; ++b) dst[b] = uint8_t(crc >> (8 * b));
      if (value_out) {
        value_out[0] = crc;
        if (stored)
          value_out[1] = uint32_t(stored[0]) | (uint32_t(stored[1]) << 8) | (uint32_t(stored[2]) << 16) |
                         (uint32_t(stored[3]) << 24);
      }
    }
  }
}

struct Head {
  uint8_t bytes[29];  // magic .. nscales (everything before the scale)
};

__global__ void pack_kernel(const int8_t* __restrict__ codes, int64_t ld, int64_t R, int64_t K, int bits, Head head,
                            const float* __restrict__ scale, uint8_t* __restrict__ out) {
  const int64_t count = R * K;
  const int64_t nbytes = bits == 8 ? count : (count + 1) / 2;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid < 29) out[tid] = head.bytes[tid];
  if (tid == 0) {
    uint32_t s;
    memcpy(&s, scale, 4);
    for (int b = 0; b < 4; ++b) out[29 + b] = uint8_t(s >> (8 * b));
  }
  uint8_t* pay = out + 33;
  for (int64_t j = tid; j < nbytes; j += int64_t(gridDim.x) * blockDim.x) {
    if (bits == 8) {
      const int64_t k = j / R, r = j - k * R;
      pay[j] = uint8_t(codes[r * ld + k]);
    } else {
      uint8_t v = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t e = 2 * j + h;
        if (e < count) {
          const int64_t k = e / R, r = e - k * R;
          v |= uint8_t((uint32_t(codes[r * ld + k]) & 0xFu) << (4 * h));
        }
      }
      pay[j] = v;
    }
  }
}

// int8 payload transposes through a 64 x 64 shared tile: dst[c * ld_dst + r] =
// src[r * ld_src + c] for r < rows, c < cols (rows_out > rows zero-fills the
// destination's padding columns).  Every global access is a warp-wide run of
// 32 consecutive bytes, so the container's unaligned payload (byte 33 on) needs
// no special case.  CHECK: first source byte 0x80 (-128, outside the symmetric
// int8 range) -> *bad (atomicMin).
template <bool CHECK>
__global__ void __launch_bounds__(256) transpose8_kernel(const uint8_t* __restrict__ src, int64_t ld_src, int64_t rows,
                                                         int64_t cols, int64_t rows_out, uint8_t* __restrict__ dst,
                                                         int64_t ld_dst, unsigned long long* bad) {
  __shared__ uint8_t tile[64][65];
  const int64_t r0 = int64_t(blockIdx.y) * 64, c0 = int64_t(blockIdx.x) * 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = warp * 8 + i;
    const int64_t r = r0 + rr;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t c = c0 + h * 32 + lane;
      uint8_t v = 0;
      if (r < rows && c < cols) {
        v = __ldg(src + r * ld_src + c);
        if (CHECK && v == 0x80) atomicMin(bad, (unsigned long long)(r * ld_src + c));
      }
      tile[rr][h * 32 + lane] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int cc = warp * 8 + i;
    const int64_t c = c0 + cc;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = r0 + h * 32 + lane;
      if (c < cols && r < rows_out) dst[c * ld_dst + r] = tile[h * 32 + lane][cc];
    }
  }
}

// payload range check (int8 -128 / int4 -8 are outside the symmetric range),
// first offending payload byte -> *bad (atomicMin), and the transpose back
__global__ void unpack_kernel(const uint8_t* __restrict__ pay, int64_t R, int64_t K, int bits, int8_t* __restrict__ codes,
                              int64_t ld, unsigned long long* bad) {
  const int64_t count = R * K;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x) {
    int v;
    int64_t at;
    if (bits == 8) {
      v = int(int8_t(pay[e]));
      at = e;
      if (v == -128) atomicMin(bad, (unsigned long long)at);
    } else {
      const uint8_t b = pay[e >> 1];
      int nib = (e & 1) ? (b >> 4) : (b & 0xF);
      v = nib >= 8 ? nib - 16 : nib;
      at = e >> 1;
      if (v == -8) atomicMin(bad, (unsigned long long)at);
    }
    const int64_t k = e / R, r = e - k * R;
    if (codes) codes[r * ld + k] = int8_t(v);
  }
}

int crc_into(const uint8_t* buf, int64_t n, uint32_t* ws, uint8_t* dst, uint32_t* value_out, const uint8_t* stored,
             cudaStream_t st) {
  int64_t nch = 1;
  while (nch * kChunk16 < n) nch <<= 1;
  const int64_t vpad = nch * kChunk16 - n;
  int64_t grid = nch < int64_t(num_sms()) * 8 ? nch : int64_t(num_sms()) * 8;
  crc_chunks16_kernel<<<int(grid), 256, 0, st>>>(buf, n, vpad, nch, (reinterpret_cast<uintptr_t>(buf) & 15) == 0, ws);
  crc_finish16_kernel<<<1, 1024, 0, st>>>(ws, nch, n, dst, value_out, stored);
  return int(cudaGetLastError());
}

}  // namespace

size_t acbp_ws_bytes(int64_t nbytes) {
  int64_t nch = 1;
  while (nch * kChunk16 < nbytes) nch <<= 1;
  return size_t(nch * 4 + 64);
}

int acbp_pack(const int8_t* codes, int64_t ld, int64_t R, int64_t K, int bits, const uint8_t* head29,
              const float* scale, uint8_t* out, int64_t total, void* ws, cudaStream_t st) {
  if (!ensure_tables()) return int(cudaErrorInitializationError);
  Head h;
  memcpy(h.bytes, head29, 29);
  const int64_t nbytes = bits == 8 ? R * K : (R * K + 1) / 2;
  int64_t grid = (nbytes + 255) / 256;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  if (grid < 1) grid = 1;
  if (bits == 8) {
    pack_kernel<<<1, 64, 0, st>>>(codes, ld, 0, 0, bits, h, scale, out);  // header + scale only
    if (R * K > 0 && (R + 63) / 64 <= 65535)
      transpose8_kernel<false><<<dim3(unsigned((K + 63) / 64), unsigned((R + 63) / 64)), 256, 0, st>>>(
          reinterpret_cast<const uint8_t*>(codes), ld, R, K, R, out + 33, R, nullptr);
    else if (R * K > 0)
      pack_kernel<<<int(grid), 256, 0, st>>>(codes, ld, R, K, bits, h, scale, out);
  } else {
    pack_kernel<<<int(grid), 256, 0, st>>>(codes, ld, R, K, bits, h, scale, out);
  }
  return crc_into(out, total - 4, static_cast<uint32_t*>(ws), out + total - 4, nullptr, nullptr, st);
}

int acbp_check_and_unpack(const uint8_t* buf, int64_t total, int64_t R, int64_t K, int bits, int8_t* codes, int64_t ld,
                          float* scale_out, void* ws, int64_t* bad_offset, bool* crc_ok, cudaStream_t st) {
  if (!ensure_tables()) return int(cudaErrorInitializationError);
  // ws: [0, 8) first bad payload byte, [8, 16) computed / stored CRC, [64, ...) chunk CRCs
  uint8_t* w = static_cast<uint8_t*>(ws);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(w);
  uint32_t* crc_val = reinterpret_cast<uint32_t*>(w + 8);
  uint32_t* chunks = reinterpret_cast<uint32_t*>(w + 64);
  cudaMemsetAsync(bad, 0xFF, 8, st);
  const int64_t count = R * K;
  int64_t grid = (count + 255) / 256;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  if (grid < 1) grid = 1;
  // the payload is (K, R) C order; codes are (R, ld) K-major, padding columns zeroed
  if (count > 0 && bits == 8 && codes && (K + 63) / 64 <= 65535 && (ld + 63) / 64 <= 65535)
    transpose8_kernel<true><<<dim3(unsigned((R + 63) / 64), unsigned((ld + 63) / 64)), 256, 0, st>>>(
        buf + 33, R, K, R, ld, reinterpret_cast<uint8_t*>(codes), ld, bad);
  else if (count > 0)
    unpack_kernel<<<int(grid), 256, 0, st>>>(buf + 33, R, K, bits, codes, ld, bad);
  if (scale_out) cudaMemcpyAsync(scale_out, buf + 29, 4, cudaMemcpyDeviceToDevice, st);
  int e = crc_into(buf, total - 4, chunks, nullptr, crc_val, buf + total - 4, st);
  if (e) return e;
  uint32_t res[4];  // bad offset (2 words), computed CRC, stored CRC: one copy back
  cudaMemcpyAsync(res, w, 16, cudaMemcpyDeviceToHost, st);
  e = int(cudaStreamSynchronize(st));
  if (e) return e;
  const unsigned long long hb = (unsigned long long)res[0] | ((unsigned long long)res[1] << 32);
  *bad_offset = hb == ~0ull ? -1 : int64_t(hb);
  *crc_ok = res[2] == res[3];
  return 0;
}

}  // namespace hlq
