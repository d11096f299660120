// device_crc.cuh — zlib-compatible CRC-32 (crc32_of, format.cpp:163-166) for
// sm_100a, split into independent chunks and recombined with GF(2) algebra:
//
//   crc(M) = XOR_i  x^(8 * bytes_after_i) (x) crc(chunk_i)     (mod P)
//
// (the closed form of zlib's crc32_combine applied left to right), so every
// lane / CTA can CRC its own bytes and fold the result into one 32-bit XOR
// accumulator per page with atomicXor — no ordering between chunks.
#pragma once

#include <cstdint>

namespace pcp {
namespace crc {

constexpr uint32_t kPoly = 0xEDB88320u;

__host__ __device__ inline uint32_t table_entry(uint32_t i) {
  uint32_t c = i;
  for (int k = 0; k < 8; ++k) c = (c & 1) ? kPoly ^ (c >> 1) : c >> 1;
  return c;
}

// a (x) b mod P, reflected (zlib multmodp).
__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

// x^(2^k) mod P for k = 0..31 (zlib x2n_table), in constant memory.
struct X2N {
  uint32_t v[32];
};

__host__ inline X2N make_x2n() {
  X2N t;
  uint32_t p = 1u << 30;  // x^1
  t.v[0] = p;
  for (int n = 1; n < 32; ++n) t.v[n] = p = multmodp(p, p);
  return t;
}

// x^(8n) mod P (zlib x2nmodp(n, 3)).
__device__ inline uint32_t x8n(const uint32_t* x2n, uint64_t n) {
  uint32_t p = 1u << 31;
  unsigned k = 3;
  while (n) {
    if (n & 1) p = multmodp(x2n[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}

// Standard CRC of bytes p[0..n) (init/xorout 0xFFFFFFFF), table in smem.
__device__ inline uint32_t bytes(const uint32_t* tab, const uint8_t* p, uint64_t n) {
  uint32_t c = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < n; ++i) c = tab[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// Same over aligned 4-byte words (bytes up to the first word boundary and
// after the last one one at a time).  Words are loaded kBatch at a time
// ahead of the table chain, so a chunk in global memory exposes the load
// latency once per batch instead of once per word.
constexpr int kBatch = 16;

__device__ __forceinline__ uint32_t word_step(const uint32_t* tab, uint32_t c, uint32_t w) {
  c ^= w;
  c = tab[c & 0xFF] ^ (c >> 8);
  c = tab[c & 0xFF] ^ (c >> 8);
  c = tab[c & 0xFF] ^ (c >> 8);
  return tab[c & 0xFF] ^ (c >> 8);
}

__device__ inline uint32_t bytes_words(const uint32_t* tab, const uint8_t* p, uint64_t n) {
  uint32_t c = 0xFFFFFFFFu;
  uint64_t i = 0;
  const uint64_t head = (4 - ((uintptr_t)p & 3)) & 3;
  for (; i < head && i < n; ++i) c = tab[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  for (; i + 4 * kBatch <= n; i += 4 * kBatch) {
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(p + i);
    uint32_t v[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) v[b] = wp[b];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) c = word_step(tab, c, v[b]);
  }
  for (; i + 4 <= n; i += 4) c = word_step(tab, c, *reinterpret_cast<const uint32_t*>(p + i));
  for (; i < n; ++i) c = tab[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

__device__ inline uint32_t warp_xor(uint32_t v) {
  for (int o = 16; o > 0; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Chunk size of the parallel CRC.  Chunks are aligned to the END of a
// range, so chunk k sits 256*k bytes before it and its shift is the constant
// x^(8*256*k), read from a host-built table (kShiftEntries entries).
constexpr uint32_t kChunk = 256;
constexpr uint32_t kShiftEntries = 8192;  // ranges up to 2 MiB use the table

__device__ inline uint32_t chunk_shift(const uint32_t* shift_tab, const uint32_t* x2n,
                                       uint64_t k) {
  return k < kShiftEntries ? shift_tab[k] : x8n(x2n, k * kChunk);
}

// CTA-cooperative CRC contribution of bytes p[0..n), which sit `after`
// bytes before the end of the page:  x^(8*after) (x) crc(p[0..n)).
// Returns the value on thread 0 (others: 0).  `red` is >= 32 words of smem.
// Four full kChunk-byte chunks (same alignment: they sit multiples of kChunk
// apart) in one pass: four independent table chains interleaved, so the
// shared-memory lookup latency is paid once per four bytes instead of once
// per byte.  Returns the four standard CRCs.
__device__ __forceinline__ void chunks4(const uint32_t* tab, const uint8_t* const (&p)[4], uint32_t (&out)[4]) {
  uint32_t c[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
  const uint32_t head = (4 - ((uintptr_t)p[0] & 3)) & 3;
  for (uint32_t i = 0; i < head; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = tab[(c[q] ^ p[q][i]) & 0xFF] ^ (c[q] >> 8);
  const uint32_t nw = (kChunk - head) / 4;
  for (uint32_t w0 = 0; w0 < nw; w0 += 4) {
    uint32_t v[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        v[q][b] = w0 + b < nw ? reinterpret_cast<const uint32_t*>(p[q] + head)[w0 + b] : 0u;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (w0 + b >= nw) break;
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] ^= v[q][b];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = tab[c[q] & 0xFF] ^ (c[q] >> 8);
    }
  }
  for (uint32_t i = head + 4 * nw; i < kChunk; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = tab[(c[q] ^ p[q][i]) & 0xFF] ^ (c[q] >> 8);
#pragma unroll
  for (int q = 0; q < 4; ++q) out[q] = c[q] ^ 0xFFFFFFFFu;
}

// The shift table buffer carries, after its kShiftEntries chunk shifts,
// byte-sliced multiplication tables by S = x^(8 * kChunk * stride) for the
// chunk strides the kernels use (lane stride 32, CTA strides 256 and 512):
// S (x) v = T[0][v & 255] ^ T[1][v >> 8 & 255] ^ T[2][..] ^ T[3][v >> 24]
// (multiplication is linear in v), four cached loads instead of a 32-step
// bit loop.
constexpr uint32_t kMulStrides[3] = {32, 256, 512};
constexpr uint32_t kShiftTabWords = kShiftEntries + 3 * 1024;

__device__ __forceinline__ const uint32_t* stride_mul_tab(const uint32_t* shift_tab, uint64_t stride) {
  const int i = stride == 32 ? 0 : stride == 256 ? 1 : stride == 512 ? 2 : -1;  // kMulStrides
  return i < 0 ? nullptr : shift_tab + kShiftEntries + 1024 * i;
}

__device__ __forceinline__ uint32_t mul_tab(const uint32_t* T, uint32_t v) {
  return __ldg(T + (v & 255u)) ^ __ldg(T + 256 + ((v >> 8) & 255u)) ^ __ldg(T + 512 + ((v >> 16) & 255u)) ^
         __ldg(T + 768 + (v >> 24));
}

// Ranges beyond the shift table (S3DIS rooms: 24 MB): chunk k_j = first +
// j * stride has shift x^(8*kChunk*first) (x) S^j, so the thread folds its
// chunks Horner-style from the highest j down (acc = S (x) acc ^ crc_j: one
// table multiply per chunk) and applies its first chunk's shift once at the
// end, instead of rebuilding x^(8n) per chunk.  Out of line: the inlined
// short-range path below stays as small as it was (k_cloud's FPS registers).
static __device__ __noinline__ uint32_t strided_chunks_long(const uint32_t* tab, const uint32_t* x2n,
                                                     const uint32_t* shift_tab, const uint8_t* p,
                                                     uint64_t n, uint64_t first, uint64_t stride) {
  const uint64_t nchunks = (n + kChunk - 1) / kChunk;
  const uint64_t full = n / kChunk;
  if (first >= nchunks) return 0;
  const uint32_t* T = stride_mul_tab(shift_tab, stride);
  const uint32_t S = T ? 0u : x8n(x2n, stride * kChunk);
  auto mulS = [&](uint32_t v) -> uint32_t { return T ? mul_tab(T, v) : multmodp(S, v); };
  int64_t j = (int64_t)((nchunks - 1 - first) / stride);
  uint32_t acc = 0;
  for (; j >= 0 && first + (uint64_t)j * stride >= full; --j) {  // the short chunk at the range start
    const uint64_t e = n - (first + (uint64_t)j * stride) * kChunk;
    const uint64_t s = e > kChunk ? e - kChunk : 0;
    acc = mulS(acc) ^ bytes_words(tab, p + s, e - s);
  }
  for (; j >= 3; j -= 4) {
    const uint8_t* ps[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ps[q] = p + (n - (first + (uint64_t)(j - q) * stride + 1) * kChunk);
    uint32_t r[4];
    chunks4(tab, ps, r);
#pragma unroll
    for (int q = 0; q < 4; ++q) acc = mulS(acc) ^ r[q];
  }
  for (; j >= 0; --j)
    acc = mulS(acc) ^ bytes_words(tab, p + (n - (first + (uint64_t)j * stride + 1) * kChunk), kChunk);
  return multmodp(chunk_shift(shift_tab, x2n, first), acc);
}

// XOR of shifted chunk CRCs for chunks k = first, first+stride, ... of a
// range of n bytes (chunks aligned to its end): four full chunks at a time,
// the rest (incl. the short chunk at the range start) one by one; one
// independent product per chunk (ILP across chunks).
__device__ __forceinline__ uint32_t strided_chunks(const uint32_t* tab, const uint32_t* x2n,
                                                   const uint32_t* shift_tab, const uint8_t* p,
                                                   uint64_t n, uint64_t first, uint64_t stride) {
  const uint64_t nchunks = (n + kChunk - 1) / kChunk;
  if (nchunks > kShiftEntries) return strided_chunks_long(tab, x2n, shift_tab, p, n, first, stride);
  const uint64_t full = n / kChunk;  // chunks 0..full-1 are full-size
  uint32_t c = 0;
  uint64_t k = first;
  for (; k + 3 * stride < full; k += 4 * stride) {
    const uint8_t* ps[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ps[q] = p + (n - (k + q * stride + 1) * kChunk);
    uint32_t r[4];
    chunks4(tab, ps, r);
#pragma unroll
    for (int q = 0; q < 4; ++q) c ^= multmodp(chunk_shift(shift_tab, x2n, k + q * stride), r[q]);
  }
  for (; k < nchunks; k += stride) {
    const uint64_t e = n - k * kChunk;
    const uint64_t s = e > kChunk ? e - kChunk : 0;
    c ^= multmodp(chunk_shift(shift_tab, x2n, k), bytes_words(tab, p + s, e - s));
  }
  return c;
}

__device__ inline uint32_t cta_range(const uint32_t* tab, const uint32_t* x2n,
                                     const uint32_t* shift_tab, const uint8_t* p,
                                     uint64_t n, uint64_t after, uint32_t* red) {
  const int t = threadIdx.x, nt = blockDim.x;
  uint32_t c = strided_chunks(tab, x2n, shift_tab, p, n, t, nt);
  c = warp_xor(c);
  if ((t & 31) == 0) red[t >> 5] = c;
  __syncthreads();
  uint32_t r = 0;
  if (t < 32) {
    r = (t < (nt + 31) / 32) ? red[t] : 0;
    r = warp_xor(r);
    if (t == 0 && after) r = multmodp(x8n(x2n, after), r);
  }
  __syncthreads();
  return t == 0 ? r : 0;
}

// Warp-cooperative version (no block barriers): used by the standalone page
// CRC kernel, where one warp owns one window of a page.
__device__ inline uint32_t warp_range(const uint32_t* tab, const uint32_t* x2n,
                                      const uint32_t* shift_tab, const uint8_t* p,
                                      uint64_t n, uint64_t after) {
  const int lane = threadIdx.x & 31;
  uint32_t c = strided_chunks(tab, x2n, shift_tab, p, n, lane, 32);
  c = warp_xor(c);
  if (after) c = multmodp(x8n(x2n, after), c);
  return c;
}

}  // namespace crc
}  // namespace pcp
