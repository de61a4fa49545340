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
// right-aligned in a power-of-two number of 4 KiB chunks (leading zeros keep a
// zero-state CRC at zero), so every combine is between equal power-of-two
// blocks: each CTA reduces a chunk (256 threads x 16 bytes, then an 8-level
// shift-and-xor tree), one 1024-thread CTA folds the chunk CRCs, and the
// 0xFFFFFFFF initial register enters as shift(0xFFFFFFFF, n).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "hlq_internal.h"

namespace hlq {

namespace {

constexpr int kChunk = 4096;
constexpr int kPiece = 16;
constexpr int kPow = 40;  // shift tables for 2^j bytes, j = 0..39

__device__ uint32_t g_crc_tab[256];
__device__ uint32_t g_crc_pow[kPow][4][256];

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
  if (cudaMemcpyToSymbol(g_crc_tab, host_tab, sizeof(host_tab)) != cudaSuccess) return false;
  if (cudaMemcpyToSymbol(g_crc_pow, pw, sizeof(pw)) != cudaSuccess) return false;
  done[dev] = true;
  return true;
}

__device__ __forceinline__ uint32_t shift_pow(uint32_t x, int j) {
  return __ldg(&g_crc_pow[j][0][x & 0xFFu]) ^ __ldg(&g_crc_pow[j][1][(x >> 8) & 0xFFu]) ^
         __ldg(&g_crc_pow[j][2][(x >> 16) & 0xFFu]) ^ __ldg(&g_crc_pow[j][3][x >> 24]);
}

// The message is right-aligned in a virtual buffer of nch (a power of two)
// 4 KiB chunks: leading zero bytes leave a zero-state CRC at zero, so every
// chunk is full and the tree below combines equal-sized blocks only.
__global__ void __launch_bounds__(256) crc_chunks_kernel(const uint8_t* __restrict__ buf, int64_t n, int64_t vpad,
                                                         uint32_t* __restrict__ out) {
  __shared__ uint32_t part[256];
  __shared__ uint8_t data[kChunk];
  const int64_t c0 = int64_t(blockIdx.x) * kChunk - vpad;  // real offset of this chunk's first byte
  for (int i = threadIdx.x; i < kChunk; i += 256) {          // coalesced stage of the chunk
    const int64_t o = c0 + i;
    data[i] = (o >= 0 && o < n) ? buf[o] : 0;
  }
  __syncthreads();
  uint32_t r = 0;
  const uint8_t* p = data + threadIdx.x * kPiece;
#pragma unroll
  for (int i = 0; i < kPiece; ++i) r = g_crc_tab[(r ^ p[i]) & 0xFFu] ^ (r >> 8);
  part[threadIdx.x] = r;
  __syncthreads();
#pragma unroll 1
  for (int j = 0; j < 8; ++j) {  // combine pieces of 16 << j bytes pairwise: shift by 2^(4+j)
    const int stride = 1 << j;
    if ((threadIdx.x & (2 * stride - 1)) == 0)
      part[threadIdx.x] = shift_pow(part[threadIdx.x], 4 + j) ^ part[threadIdx.x + stride];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = part[0];
}

// one CTA: each thread folds nch/1024 consecutive chunk CRCs, then a tree;
// zlib crc32 = raw ^ shift(0xFFFFFFFF, n) ^ 0xFFFFFFFF
__global__ void __launch_bounds__(1024) crc_finish_kernel(const uint32_t* __restrict__ chunks, int64_t nch, int64_t n,
                                                          uint8_t* dst, uint32_t* value_out) {
  __shared__ uint32_t part[1024];
  const int64_t per = nch >= 1024 ? nch / 1024 : 1;
  const int active = int(nch >= 1024 ? 1024 : nch);
  uint32_t r = 0;
  if (int(threadIdx.x) < active)
    for (int64_t c = threadIdx.x * per; c < (threadIdx.x + 1) * per; ++c) r = shift_pow(r, 12) ^ chunks[c];
  part[threadIdx.x] = r;
  __syncthreads();
  int lg = 12;  // log2 bytes of one thread's block
  for (int64_t p = per; p > 1; p >>= 1) ++lg;
  for (int stride = 1; stride < active; stride <<= 1, ++lg) {
    if ((threadIdx.x & (2 * stride - 1)) == 0 && int(threadIdx.x) + stride < active)
      part[threadIdx.x] = shift_pow(part[threadIdx.x], lg) ^ part[threadIdx.x + stride];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint32_t init = 0xFFFFFFFFu;
    for (int j = 0; j < kPow; ++j)
      if ((n >> j) & 1) init = shift_pow(init, j);
    const uint32_t crc = part[0] ^ init ^ 0xFFFFFFFFu;
    if (dst)
      for (int b = 0; b < 4; ++b) dst[b] = uint8_t(crc >> (8 * b));
    if (value_out) *value_out = crc;
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

// int8 payload: (R, K) K-major codes -> (K, R) C-order bytes through a 64 x 64
// shared tile (both sides coalesced); the int4 path keeps pack_kernel
__global__ void __launch_bounds__(256) pack8_tiled_kernel(const int8_t* __restrict__ codes, int64_t ld, int64_t R,
                                                          int64_t K, uint8_t* __restrict__ pay) {
  __shared__ uint8_t tile[64][65];
  const int64_t r0 = int64_t(blockIdx.y) * 64, k0 = int64_t(blockIdx.x) * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  for (int i = ty; i < 64; i += 4) {
    const int64_t r = r0 + i, k = k0 + tx;
    tile[i][tx] = (r < R && k < K) ? uint8_t(codes[r * ld + k]) : 0;
  }
  __syncthreads();
  for (int i = ty; i < 64; i += 4) {
    const int64_t k = k0 + i, r = r0 + tx;
    if (k < K && r < R) pay[k * R + r] = tile[tx][i];
  }
}

__global__ void __launch_bounds__(256) unpack8_tiled_kernel(const uint8_t* __restrict__ pay, int64_t R, int64_t K,
                                                            int8_t* __restrict__ codes, int64_t ld,
                                                            unsigned long long* bad) {
  __shared__ uint8_t tile[64][65];
  const int64_t r0 = int64_t(blockIdx.y) * 64, k0 = int64_t(blockIdx.x) * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  for (int i = ty; i < 64; i += 4) {
    const int64_t k = k0 + i, r = r0 + tx;
    uint8_t v = 0;
    if (k < K && r < R) {
      v = pay[k * R + r];
      if (v == 0x80) atomicMin(bad, (unsigned long long)(k * R + r));
    }
    tile[tx][i] = v;
  }
  __syncthreads();
  for (int i = ty; i < 64; i += 4) {
    const int64_t r = r0 + i, k = k0 + tx;
    if (r < R && k < K) codes[r * ld + k] = int8_t(tile[i][tx]);
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

int crc_into(const uint8_t* buf, int64_t n, uint32_t* ws, uint8_t* dst, uint32_t* value_out, cudaStream_t st) {
  int64_t nch = 1;
  while (nch * kChunk < n) nch <<= 1;
  const int64_t vpad = nch * kChunk - n;
  crc_chunks_kernel<<<int(nch), 256, 0, st>>>(buf, n, vpad, ws);
  crc_finish_kernel<<<1, 1024, 0, st>>>(ws, nch, n, dst, value_out);
  return int(cudaGetLastError());
}

}  // namespace

size_t acbp_ws_bytes(int64_t nbytes) {
  int64_t nch = 1;
  while (nch * kChunk < nbytes) nch <<= 1;
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
      pack8_tiled_kernel<<<dim3(unsigned((K + 63) / 64), unsigned((R + 63) / 64)), 256, 0, st>>>(codes, ld, R, K,
                                                                                                  out + 33);
    else if (R * K > 0)
      pack_kernel<<<int(grid), 256, 0, st>>>(codes, ld, R, K, bits, h, scale, out);
  } else {
    pack_kernel<<<int(grid), 256, 0, st>>>(codes, ld, R, K, bits, h, scale, out);
  }
  return crc_into(out, total - 4, static_cast<uint32_t*>(ws), out + total - 4, nullptr, st);
}

int acbp_check_and_unpack(const uint8_t* buf, int64_t total, int64_t R, int64_t K, int bits, int8_t* codes, int64_t ld,
                          float* scale_out, void* ws, int64_t* bad_offset, bool* crc_ok, cudaStream_t st) {
  if (!ensure_tables()) return int(cudaErrorInitializationError);
  uint8_t* w = static_cast<uint8_t*>(ws);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(w);
  uint32_t* crc_val = reinterpret_cast<uint32_t*>(w + 8);
  uint32_t* chunks = reinterpret_cast<uint32_t*>(w + 64);
  cudaMemsetAsync(bad, 0xFF, 8, st);
  const int64_t count = R * K;
  int64_t grid = (count + 255) / 256;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  if (grid < 1) grid = 1;
  if (count > 0 && bits == 8 && codes && (R + 63) / 64 <= 65535)
    unpack8_tiled_kernel<<<dim3(unsigned((K + 63) / 64), unsigned((R + 63) / 64)), 256, 0, st>>>(buf + 33, R, K,
                                                                                                  codes, ld, bad);
  else if (count > 0)
    unpack_kernel<<<int(grid), 256, 0, st>>>(buf + 33, R, K, bits, codes, ld, bad);
  if (scale_out) cudaMemcpyAsync(scale_out, buf + 29, 4, cudaMemcpyDeviceToDevice, st);
  int e = crc_into(buf, total - 4, chunks, nullptr, crc_val, st);
  if (e) return e;
  unsigned long long hb = 0;
  uint32_t hc = 0;
  uint8_t stored[4];
  cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&hc, crc_val, 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(stored, buf + total - 4, 4, cudaMemcpyDeviceToHost, st);
  e = int(cudaStreamSynchronize(st));
  if (e) return e;
  *bad_offset = hb == ~0ull ? -1 : int64_t(hb);
  const uint32_t sv = uint32_t(stored[0]) | (uint32_t(stored[1]) << 8) | (uint32_t(stored[2]) << 16) |
                      (uint32_t(stored[3]) << 24);
  *crc_ok = sv == hc;
  return 0;
}

}  // namespace hlq
