// page_encode.cu — PcRecord page encoder on the B200:
// encode_block_page / encode_scalar_page (format.cpp:198-274) for a batch of
// pages, byte-identical to the reference: XOR-delta columns, the greedy
// LZ4 block compressor (lz4_block.cpp:33-103), the stored-raw fallback when
// LZ4 does not shrink the page, and the payload CRC-32.
//
// The reference compressor is one serial greedy parse per page whose hash
// table holds, for every 16-bit hash, the last position the parse VISITED
// (match interiors are skipped).  Here everything around that parse is
// parallel and the parse itself does O(1) cheap work per position:
//
//   delta   thread per word: w[i] ^= w[i-1] inside every delta column
//   hash    thread per position p < n-12: (hash(read32(p)), p)
//   sort    segmented stable radix sort by hash (CUB) per page
//   prev    prev[p] = the previous position with the same hash (any, visited
//           or not) -> the table lookup becomes a walk down prev[] past
//           positions inside emitted matches (a visited bitmap)
//   parse   one warp per page: the reference's loop with its hash table,
//           32 positions speculated per step (candidates inside the step's
//           literal run come from prev[]; the first matching lane wins);
//           records the sequences
//   emit    CTA per page: token/length bytes and literals in parallel at
//           offsets from a block scan over the sequences' output sizes
//   crc     the existing CTA-cooperative CRC over the chosen payload
#include <cuda_runtime.h>

#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <cstdint>

#include "device_crc.cuh"
#include "page_encode.h"

namespace pcp {

__constant__ crc::X2N c_x2n_enc;

namespace {

constexpr uint32_t kMinMatch = 4, kLastLiterals = 5, kMfLimit = 12, kMaxOffset = 65535;
constexpr uint32_t kNone = 0xffffffffu;

__device__ __forceinline__ uint32_t read32u(const uint8_t* p) {  // unaligned
  return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
}
__device__ __forceinline__ uint32_t hash32(uint32_t v) { return (v * 2654435761u) >> 16; }

// XOR-delta encode (format.cpp:168-181, width 4) of every column, in place on
// the work copy (reads the raw page, writes work: no ordering hazard).
__global__ void k_enc_delta(const uint8_t* raw, uint8_t* work, const EncPage* pages, const EncColumn* cols,
                            uint32_t n_cols) {
  for (uint32_t c = blockIdx.x; c < n_cols; c += gridDim.x) {
    const EncColumn col = cols[c];
    const EncPage pg = pages[col.page];
    const uint8_t* in = raw + pg.raw_off + col.off;
    uint8_t* out = work + pg.raw_off + col.off;
    const uint64_t words = col.len / 4;
    for (uint64_t i = 1 + threadIdx.x; i < words; i += blockDim.x) {
      const uint32_t x = read32u(in + 4 * i) ^ read32u(in + 4 * (i - 1));
      out[4 * i] = (uint8_t)x;
      out[4 * i + 1] = (uint8_t)(x >> 8);
      out[4 * i + 2] = (uint8_t)(x >> 16);
      out[4 * i + 3] = (uint8_t)(x >> 24);
    }
  }
}

// (hash, position) for every position a parse can visit (p < n - 12).
__global__ void k_enc_hash(const uint8_t* work, const EncPage* pages, uint32_t n_pages, uint32_t* keys,
                           uint32_t* vals) {
  for (uint32_t pi = blockIdx.y; pi < n_pages; pi += gridDim.y) {
    const EncPage pg = pages[pi];
    const uint64_t np = pg.raw_len > kMfLimit ? pg.raw_len - kMfLimit : 0;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (uint64_t)gridDim.x * blockDim.x) {
      keys[pg.hash_off + p] = hash32(read32u(work + pg.raw_off + p));
      vals[pg.hash_off + p] = (uint32_t)p;
    }
  }
}

// prev[p] = the previous position (in the page) with the same hash, or none.
__global__ void k_enc_prev(const uint32_t* keys, const uint32_t* vals, const EncPage* pages, uint32_t n_pages,
                           uint32_t* prev) {
  for (uint32_t pi = blockIdx.y; pi < n_pages; pi += gridDim.y) {
    const EncPage pg = pages[pi];
    const uint64_t np = pg.raw_len > kMfLimit ? pg.raw_len - kMfLimit : 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t g = pg.hash_off + i;
      prev[pg.hash_off + vals[g]] = (i > 0 && keys[g - 1] == keys[g]) ? vals[g - 1] : kNone;
    }
  }
}

// The reference parse (lz4_block.cpp:75-99), one WARP per page, with the
// reference's hash table (last VISITED position per 16-bit hash, stored +1
// so 0 = empty) in global memory.  Lanes speculate on 32 consecutive
// positions ip..ip+31: if no match starts before ip+k, positions ip..ip+k-1
// are visited too, so lane k's candidate is its previous same-hash position
// when that lies in [ip, ip+k) (prev[]), else the table entry.  The first
// lane whose candidate matches is where the serial parse takes its match
// (ballot); positions ip..ip+k are inserted (atomicMax: later positions win).
// Match extension compares 32 bytes per step.
__global__ void k_enc_parse(const uint8_t* work, const EncPage* pages, uint32_t n_pages, const uint32_t* prev,
                            const uint32_t* hashes, uint32_t* table, EncSeq* seqs, uint32_t* n_seqs) {
  const uint32_t pi = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (pi >= n_pages) return;  // warp-uniform
  const EncPage pg = pages[pi];
  const uint8_t* src = work + pg.raw_off;
  const uint64_t n = pg.raw_len;
  const uint32_t* pv = prev + pg.hash_off;
  const uint32_t* hs = hashes + pg.hash_off;
  uint32_t* tab = table + (uint64_t)pi * 65536;
  EncSeq* out = seqs + pg.seq_off;
  uint32_t ns = 0;
  uint64_t ip = 0, anchor = 0;
  if (n > kMfLimit) {
    const uint64_t match_limit = n - kMfLimit, end_limit = n - kLastLiterals;
    while (ip < match_limit) {
      const uint64_t p = ip + lane;
      bool hit = false;
      uint32_t cand = kNone, h = 0;
      if (p < match_limit) {
        h = hs[p];
        const uint32_t pp = pv[p];
        if (pp != kNone && pp >= ip) {
          cand = pp;  // visited in this speculative literal run
        } else {
          const uint32_t t = tab[h];
          cand = t ? t - 1 : kNone;
        }
        hit = cand != kNone && p - cand <= kMaxOffset && read32u(src + cand) == read32u(src + p);
      }
      const uint32_t hits = __ballot_sync(0xffffffffu, hit);
      const uint32_t valid = __ballot_sync(0xffffffffu, p < match_limit);
      const uint32_t k = hits ? __ffs(hits) - 1 : 32u;
      const uint32_t upto = min(k + (hits ? 1u : 0u), (uint32_t)__popc(valid));
      if (lane < upto) atomicMax(&tab[h], (uint32_t)p + 1u);  // table[h] = p for the visited positions
      __syncwarp();
      if (!hits) {
        ip += upto;
        continue;
      }
      const uint64_t s0 = ip + k;
      const uint32_t c0 = __shfl_sync(0xffffffffu, cand, k);
      uint64_t m = s0 + kMinMatch, r = (uint64_t)c0 + kMinMatch;
      while (true) {
        const uint64_t mm = m + lane;
        const bool eq = mm < end_limit && src[mm] == src[r + lane];
        const uint32_t neq = ~__ballot_sync(0xffffffffu, eq);
        if (neq) {
          m += __ffs(neq) - 1;
          break;
        }
        m += 32;
        r += 32;
      }
      if (lane == 0)
        out[ns] = EncSeq{(uint32_t)anchor, (uint32_t)(s0 - anchor), (uint32_t)(m - s0), (uint32_t)(s0 - c0)};
      ++ns;
      ip = m;
      anchor = ip;
    }
  }
  if (lane == 0) {
    out[ns] = EncSeq{(uint32_t)anchor, (uint32_t)(n - anchor), 0u, 0u};  // trailing literals
    n_seqs[pi] = ns + 1;
  }
}

__device__ __forceinline__ uint64_t ext_bytes(uint64_t len) {  // put_len_ext for len >= 15
  return len >= 15 ? (len - 15) / 255 + 1 : 0;
}
__device__ __forceinline__ uint64_t seq_bytes(const EncSeq& q) {
  uint64_t b = 1 + ext_bytes(q.lit_len) + q.lit_len;
  if (q.match_len) b += 2 + ext_bytes(q.match_len - kMinMatch);
  return b;
}

// CTA per page: output offsets of the sequences (block scan), headers and
// short literals by their thread, long literals by the whole CTA.
__global__ void __launch_bounds__(512) k_enc_emit(const uint8_t* work, const EncPage* pages, const EncSeq* seqs,
                                                  const uint32_t* n_seqs, uint8_t* comp, uint64_t* comp_len) {
  __shared__ uint64_t wsum[17];
  __shared__ uint64_t carry;
  const uint32_t pi = blockIdx.x;
  const EncPage pg = pages[pi];
  const EncSeq* q = seqs + pg.seq_off;
  const uint32_t ns = n_seqs[pi];
  uint8_t* dst = comp + pg.comp_off;
  const uint8_t* src = work + pg.raw_off;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b0 = 0; b0 < ns; b0 += blockDim.x) {
    const uint32_t k = b0 + threadIdx.x;
    const uint64_t sz = k < ns ? seq_bytes(q[k]) : 0;
    uint64_t inc = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if ((int)lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t acc = carry;
      for (uint32_t j = 0; j < nw; ++j) {
        const uint64_t c = wsum[j];
        wsum[j] = acc;
        acc += c;
      }
      wsum[16] = acc;
    }
    __syncthreads();
    if (k < ns) {
      uint64_t o = wsum[w] + inc - sz;
      const EncSeq s = q[k];
      const uint32_t lit = s.lit_len, ml = s.match_len ? s.match_len - kMinMatch : 0;
      dst[o++] = (uint8_t)((lit >= 15 ? 15u : lit) << 4 | (s.match_len == 0 ? 0u : (ml >= 15 ? 15u : ml)));
      if (lit >= 15) {
        uint64_t L = lit - 15;
        for (; L >= 255; L -= 255) dst[o++] = 255;
        dst[o++] = (uint8_t)L;
      }
      if (lit <= 64) {
        for (uint32_t i = 0; i < lit; ++i) dst[o + i] = src[s.lit_start + i];
      }
      o += lit;
      if (s.match_len) {
        dst[o++] = (uint8_t)(s.offset & 0xff);
        dst[o++] = (uint8_t)(s.offset >> 8);
        if (ml >= 15) {
          uint64_t L = ml - 15;
          for (; L >= 255; L -= 255) dst[o++] = 255;
          dst[o++] = (uint8_t)L;
        }
      }
    }
    // long literals of this block of sequences: copied by the whole CTA
    for (uint32_t j = 0; j < blockDim.x && b0 + j < ns; ++j) {
      const EncSeq s = q[b0 + j];
      if (s.lit_len <= 64) continue;
      // offset of sequence j's literal: recompute from the scan (thread j's exclusive offset)
      __syncthreads();
      __shared__ uint64_t lit_at;
      if (threadIdx.x == j) lit_at = wsum[j >> 5] + inc - sz + 1 + ext_bytes(s.lit_len);
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < s.lit_len; i += blockDim.x) dst[lit_at + i] = src[s.lit_start + i];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = wsum[16];
    __syncthreads();
  }
  if (threadIdx.x == 0) comp_len[pi] = carry;
}

// CRC-32 of each page's chosen payload (compressed if it shrank, else the
// post-delta raw page) -- the reference's finish_page (format.cpp:209-241).
__global__ void __launch_bounds__(256) k_enc_crc(const uint8_t* work, const uint8_t* comp, const EncPage* pages,
                                                 uint32_t n_pages, const uint64_t* comp_len,
                                                 const uint32_t* shift_tab, uint32_t* crc) {
  __shared__ uint32_t tab[256];
  __shared__ uint32_t red[32];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = crc::table_entry(i);
  __syncthreads();
  for (uint32_t pi = blockIdx.x; pi < n_pages; pi += gridDim.x) {
    const EncPage pg = pages[pi];
    const bool lz = comp_len[pi] < pg.raw_len;
    const uint8_t* p = lz ? comp + pg.comp_off : work + pg.raw_off;
    const uint64_t n = lz ? comp_len[pi] : pg.raw_len;
    const uint32_t c = crc::cta_range(tab, c_x2n_enc.v, shift_tab, p, n, 0, red);
    if (threadIdx.x == 0) crc[pi] = c;
  }
}

}  // namespace

EncScratchSizes enc_scratch_sizes(uint64_t raw_total, uint64_t hash_total, uint32_t n_pages) {
  EncScratchSizes z{};
  z.keys = 4 * hash_total;
  z.vals = 4 * hash_total;
  z.prev = 4 * hash_total;
  z.visited = 4ull * 65536 * n_pages;  // per-page hash tables
  z.seqs = sizeof(EncSeq) * (raw_total / kMinMatch + 2ull * n_pages);
  z.comp = raw_total + raw_total / 255 + 64ull * n_pages;
  size_t cub_bytes = 0;
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                           (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)hash_total,
                                           (int)n_pages, (const int*)nullptr, (const int*)nullptr, 0, 16);
  z.cub = cub_bytes + 256;
  return z;
}

cudaError_t launch_encode_pages(const EncArgs& e, cudaStream_t st) {
  static const bool x2n_done = [] {
    const crc::X2N t = crc::make_x2n();
    cudaMemcpyToSymbol(c_x2n_enc, &t, sizeof(t));
    return true;
  }();
  (void)x2n_done;
  if (!e.n_pages) return cudaSuccess;
  cudaMemcpyAsync(e.work, e.raw, e.raw_total, cudaMemcpyDeviceToDevice, st);
  if (e.n_cols) k_enc_delta<<<std::min<uint32_t>(e.n_cols, 4096), 256, 0, st>>>(e.raw, e.work, e.pages, e.cols, e.n_cols);
  cudaMemsetAsync(e.visited, 0, e.visited_bytes, st);
  const dim3 g2(64, std::min<uint32_t>(e.n_pages, 1024));
  k_enc_hash<<<g2, 256, 0, st>>>(e.work, e.pages, e.n_pages, e.keys, e.vals);
  size_t cub_bytes = e.cub_bytes;
  cudaError_t err = cub::DeviceSegmentedRadixSort::SortPairs(
      e.cub, cub_bytes, e.keys, e.keys_alt, e.vals, e.vals_alt, (int)e.hash_total, (int)e.n_pages,
      e.hash_begin, e.hash_end, 0, 16, st);
  if (err != cudaSuccess) return err;
  k_enc_prev<<<g2, 256, 0, st>>>(e.keys_alt, e.vals_alt, e.pages, e.n_pages, e.prev);
  k_enc_parse<<<(e.n_pages + 3) / 4, 128, 0, st>>>(e.work, e.pages, e.n_pages, e.prev, e.keys, e.visited,
                                                  e.seqs, e.n_seqs);
  k_enc_emit<<<e.n_pages, 512, 0, st>>>(e.work, e.pages, e.seqs, e.n_seqs, e.comp, e.comp_len);
  k_enc_crc<<<std::min<uint32_t>(e.n_pages, 1024), 256, 0, st>>>(e.work, e.comp, e.pages, e.n_pages, e.comp_len,
                                                                 e.shift_tab, e.crc);
  return cudaGetLastError();
}

}  // namespace pcp
