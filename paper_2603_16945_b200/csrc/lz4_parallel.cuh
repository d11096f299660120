// lz4_parallel.cuh — CTA-parallel decode of ONE LZ4 block (the reference
// writes one block per page, lz4_block.cpp:33-110), output byte-identical to
// lz4::decompress (lz4_block.cpp:113-156) with the same error verdicts.
//
// The token chain of an LZ4 block is serial; on the reference's pages it is
// ~1 sequence per 20 B (avg literal 16 B, match 5 B).  We
// parallelise it in four phases, all inside one CTA:
//
//  1. speculative parse: the payload is cut into CH-byte chunks; thread k
//     parses chunk k as if a token started at its first byte, marking every
//     token position it visits in a per-chunk bitmap.  LZ4 token chains are
//     self-synchronising: a chain started at a wrong byte soon lands on a
//     true token position and from then on IS the true chain.
//  2. stitch: thread k re-walks chunk k from the assumed entry (the previous
//     chunk's speculative exit) until it hits a marked position (converged),
//     verifying the exit; thread 0 then chains the true entries, re-walking
//     only chunks whose assumption failed (rare).
//  3. true parse per chunk from its verified entry: count, scan, then parse
//     again copying literals and emitting match records (all reference
//     bounds checks, in the reference's order, with the global output
//     position now known).
//  4. matches: resolved in stream order by one warp through a shared-memory
//     ring of the output (match-to-match dependency chains are thousands
//     deep on real pages, so this part is inherently sequential).
//     Overlapping copies use dst[mo+i] = dst[mo-off + i % off], the closed
//     form of the byte-wise copy.
#pragma once

#include <cstdint>

#include "pcp_internal.h"

namespace pcp {
namespace lz4p {

constexpr uint32_t kChunk = 2048;      // compressed bytes per skim window / parse chunk
constexpr uint32_t kRing = 16384;      // shared-memory output window (bytes)
constexpr uint32_t kStageTail = 64;    // staged bytes past a window for its last tokens
constexpr uint32_t kStageBytes = kChunk + kStageTail + 16;  // + alignment slack
constexpr uint32_t kSmemWords = 72 + 2 * kChunk + (2 * kStageBytes) / 4 + kChunk;
constexpr uint32_t kRingChunk = 4096;  // refill granule
constexpr uint32_t kNone = 0xFFFFFFFFu;

// Per-page scratch layout (host computes the size with scratch_bytes()).
__host__ __device__ inline uint32_t n_chunks(uint64_t pay) {
  return (uint32_t)((pay + kChunk - 1) / kChunk);
}
__host__ __device__ inline uint64_t match_capacity(uint64_t pay) { return pay / 6 + 64; }

__host__ __device__ inline uint64_t scratch_bytes(uint64_t pay) {
  const uint64_t nch = n_chunks(pay) + 1;
  return nch * (kChunk / 8)     // bitmaps
         + nch * 4 * 8          // per-chunk words (8 u32)
         + match_capacity(pay) * 16 + 256;
}

struct Scratch {
  uint32_t* bitmap;    // [nch][kChunk/32]
  uint32_t* spec_exit; // speculative exit position
  uint32_t* spec_flag; // bit0: chain ended with the last sequence, bit1: error
  uint32_t* walk_exit; // exit when walking from the assumed entry
  uint32_t* walk_flag; // bit0 last, bit1 error, bit2 converged
  uint32_t* entry;     // verified true entry
  uint32_t* cnt_out;   // output bytes of the chunk's true sequences
  uint32_t* cnt_match; // matches in the chunk
  uint32_t* base_out;  // exclusive scans
  uint32_t* m_mo;      // match output start
  uint32_t* m_ml;      // match length
  uint16_t* m_off;     // offset
  uint32_t* tokpos;    // true token positions, in stream order
};

__device__ inline Scratch carve_scratch(uint8_t* p, uint64_t pay) {
  const uint32_t nch = n_chunks(pay) + 1;
  Scratch s;
  s.bitmap = reinterpret_cast<uint32_t*>(p);
  uint32_t* w = s.bitmap + (uint64_t)nch * (kChunk / 32);
  s.spec_exit = w;
  s.spec_flag = w + nch;
  s.walk_exit = w + 2 * nch;
  s.walk_flag = w + 3 * nch;
  s.entry = w + 4 * nch;
  s.cnt_out = w + 5 * nch;
  s.cnt_match = w + 6 * nch;
  s.base_out = w + 7 * nch;
  uint32_t* m = w + 8 * nch;
  const uint64_t cap = match_capacity(pay);
  s.m_mo = m;
  s.m_ml = m + cap;
  s.m_off = reinterpret_cast<uint16_t*>(m + 2 * cap);
  s.tokpos = m + 3 * cap;
  return s;
}

// One sequence header at `ip`.  Returns false on a malformed header (same
// conditions as lz4_block.cpp:133-150 that do not need the output position).
struct Seq {
  uint32_t lit_src, lit_len, match_len, offset, next;
  bool last;
};

__device__ __forceinline__ bool parse_seq(const uint8_t* __restrict__ src, uint32_t n, uint32_t ip,
                                          Seq& s) {
  if (ip >= n) return false;
  const uint32_t token = src[ip++];
  uint32_t lit = token >> 4;
  if (lit == 15) {
    uint32_t b;
    do {
      if (ip >= n) return false;
      b = src[ip++];
      lit += b;
    } while (b == 255 && lit < 0x7fffffffu);
  }
  if ((uint64_t)ip + lit > n) return false;
  s.lit_src = ip;
  s.lit_len = lit;
  ip += lit;
  if (ip == n) {
    s.last = true;
    s.match_len = 0;
    s.offset = 0;
    s.next = n;
    return true;
  }
  if (ip + 2 > n) return false;
  s.offset = (uint32_t)src[ip] | ((uint32_t)src[ip + 1] << 8);
  ip += 2;
  if (s.offset == 0) return false;
  uint32_t ml = token & 15;
  if (ml == 15) {
    uint32_t b;
    do {
      if (ip >= n) return false;
      b = src[ip++];
      ml += b;
    } while (b == 255 && ml < 0x7fffffffu);
  }
  s.match_len = ml + 4;
  s.last = false;
  s.next = ip;
  return true;
}

// parse_seq reading bytes [c0, se) from a shared-memory copy, the rest
// (long literal runs) from global.
__device__ __forceinline__ bool parse_seq_staged(const uint8_t* buf, uint32_t c0, uint32_t se,
                                                 const uint8_t* __restrict__ src, uint32_t n,
                                                 uint32_t ip, Seq& s) {
  auto at = [&](uint32_t i) -> uint32_t { return i < se ? buf[i - c0] : src[i]; };
  if (ip >= n) return false;
  const uint32_t token = at(ip++);
  uint32_t lit = token >> 4;
  if (lit == 15) {
    uint32_t b;
    do {
      if (ip >= n) return false;
      b = at(ip++);
      lit += b;
    } while (b == 255 && lit < 0x7fffffffu);
  }
  if ((uint64_t)ip + lit > n) return false;
  s.lit_src = ip;
  s.lit_len = lit;
  ip += lit;
  if (ip == n) {
    s.last = true;
    s.match_len = 0;
    s.offset = 0;
    s.next = n;
    return true;
  }
  if (ip + 2 > n) return false;
  s.offset = at(ip) | (at(ip + 1) << 8);
  ip += 2;
  if (s.offset == 0) return false;
  uint32_t ml = token & 15;
  if (ml == 15) {
    uint32_t b;
    do {
      if (ip >= n) return false;
      b = at(ip++);
      ml += b;
    } while (b == 255 && ml < 0x7fffffffu);
  }
  s.match_len = ml + 4;
  s.last = false;
  s.next = ip;
  return true;
}

// Barrier among the fill warps only (warps 1..), id 1.
__device__ __forceinline__ void named_sync_fill(uint32_t nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ bool bit(const uint32_t* bm, uint32_t i) {
  return (bm[i >> 5] >> (i & 31)) & 1u;
}

// Walk the chain from `pos` inside chunk k until a position marked in the
// chunk's bitmap (converged), the chunk end, the last sequence or an error.
__device__ inline uint32_t walk(const uint8_t* src, uint32_t n, uint32_t k, uint32_t pos,
                                const uint32_t* bm, uint32_t& flag) {
  const uint32_t c0 = k * kChunk, c1 = min(c0 + kChunk, n);
  flag = 0;
  if (pos < c0) {  // entry assumed from an errored speculative chain
    flag = 2;
    return pos;
  }
  while (pos < c1) {
    if (bit(bm, pos - c0)) {
      flag = 4;
      return pos;
    }
    Seq s;
    if (!parse_seq(src, n, pos, s)) {
      flag = 2;
      return pos;
    }
    if (s.last) {
      flag = 1;
      return n;
    }
    pos = s.next;
  }
  return pos;
}

// Copy `len` bytes src→dst (both arbitrary alignment), one thread.
__device__ __forceinline__ void copy_bytes(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                           uint32_t len) {
  uint32_t i = 0;
  const uint32_t head = (4u - (uint32_t)((uintptr_t)dst & 3u)) & 3u;
  for (; i < head && i < len; ++i) dst[i] = src[i];
  if (((uintptr_t)(src + i) & 3u) == 0) {
    for (; i + 4 <= len; i += 4)
      *reinterpret_cast<uint32_t*>(dst + i) = *reinterpret_cast<const uint32_t*>(src + i);
  } else {
    for (; i + 4 <= len; i += 4) {
      const uint8_t* p = src + i;
      *reinterpret_cast<uint32_t*>(dst + i) =
          (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    }
  }
  for (; i < len; ++i) dst[i] = src[i];
}

// Decode one page with the whole CTA.  `ctl` is >= 8 words of shared memory.
// Returns the status (same on all threads).
__device__ inline int32_t decode_block(const uint8_t* __restrict__ src, uint32_t n,
                                       uint8_t* __restrict__ dst, uint32_t raw_len, Scratch sc,
                                       uint32_t* ctl, uint8_t* ring, long long* tm = nullptr) {
#define PCP_T(i) \
  if (tm && threadIdx.x == 0) tm[i] = clock64();
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  const uint32_t nch = n_chunks(n);

  if (t == 0) ctl[0] = 0;            // error
  if (n == 0) return kCorruptPage;   // "truncated stream" (:134)
  PCP_T(0)
  // ---- phases 1+2: skim the token chain ------------------------------------
  // Window w = compressed bytes [w*kChunk, (w+1)*kChunk).  All warps but
  // warp 0 fill the jump table of window w+1 — d[p] = distance from p to the
  // next token if a token started at p (bit 30: last sequence, bit 31:
  // malformed) — while warp 0's lane 0 walks the true chain through window w
  // with one shared-memory lookup per sequence, recording each window's
  // entry (first true token >= window start).
  {
    uint32_t* jt = ctl + 72;  // two windows of kChunk words, after ctl[0..71]
    uint8_t* wb = reinterpret_cast<uint8_t*>(jt + 2 * kChunk);  // 2 x kStageBytes bytes
    uint32_t* tbuf = jt + 2 * kChunk + (2 * kStageBytes) / 4;    // window token positions
    if (t == 0) {
      ctl[5] = 0;
      ctl[6] = 0;
    }
    // staged copy of window w: aligned 4-byte words of [c0 - sh, e) with
    // sh = misalignment of src + c0; all loads issued before the stores.
    // Readers use buf0 + sh.  Reads up to 3 bytes outside the payload on
    // either side; every byte store carries >= 16 B of slack.
    auto stage = [&](uint32_t w, uint8_t* buf0, uint32_t tid, uint32_t nthr) {
      const uint32_t c0 = w * kChunk, e = min(c0 + kChunk + kStageTail, n);
      const uintptr_t base = reinterpret_cast<uintptr_t>(src) + c0;
      const uint32_t sh = (uint32_t)(base & 3u);
      const uint32_t* g = reinterpret_cast<const uint32_t*>(base - sh);
      const uint32_t nw = (sh + (e - c0) + 3) / 4;
      uint32_t* b32 = reinterpret_cast<uint32_t*>(buf0);
      uint32_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t k = tid + u * nthr;
        v[u] = k < nw ? g[k] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t k = tid + u * nthr;
        if (k < nw) b32[k] = v[u];
      }
    };
    auto fill = [&](uint32_t w, uint32_t* tab, const uint8_t* buf0, uint32_t tid, uint32_t nthr) {
      const uint32_t c0 = w * kChunk, c1 = min(c0 + kChunk, n);
      const uint8_t* buf = buf0 + ((reinterpret_cast<uintptr_t>(src) + c0) & 3u);
      const uint32_t se = min(c0 + kChunk + kStageTail, n);
      for (uint32_t p = c0 + tid; p < c1; p += nthr) {
        Seq sq;
        uint32_t v;
        if (!parse_seq_staged(buf, c0, se, src, n, p, sq)) v = 0x80000000u;
        else if (sq.last) v = 0x40000000u | (n - p);
        else v = min(sq.next - p, 0x3FFFFFFFu);
        tab[p - c0] = v;
      }
    };
    stage(0, wb, t, nt);
    __syncthreads();
    fill(0, jt, wb, t, nt);
    if (nch > 1) stage(1, wb + kStageBytes, t, nt);
    __syncthreads();
    uint32_t pos = 0;  // walker state (thread 0)
    uint32_t err = 0, done = 0, nseq = 0;
    const uint32_t cap_seq = (uint32_t)match_capacity(n);
    for (uint32_t w = 0; w < nch; ++w) {
      if (t >= 32) {
        // fill window w+1 from its staged bytes, then stage window w+2 into
        // the buffer window w used (the walker only reads the jump table)
        if (w + 1 < nch)
          fill(w + 1, jt + ((w + 1) & 1) * kChunk, wb + ((w + 1) & 1) * kStageBytes,
               t - 32, nt - 32);
        named_sync_fill(nt - 32);
        if (w + 2 < nch) stage(w + 2, wb + (w & 1) * kStageBytes, t - 32, nt - 32);
      } else if (t == 0) {
        const uint32_t* tab = jt + (w & 1) * kChunk;
        const uint32_t c0 = w * kChunk, c1 = min(c0 + kChunk, n);
        sc.entry[w] = pos;
        uint32_t k = 0, acc = 0;
        if (!done) {
          while (pos < c1) {  // branch-free body: one LDS + one STS per token
            const uint32_t v = tab[pos - c0];
            acc |= v;
            tbuf[k++] = pos;
            pos += v & 0x3FFFFFFFu;
            if (v & 0xC0000000u) break;  // malformed or last
          }
          if (acc & 0x80000000u) err = 1;
          if (acc & 0xC0000000u) done = 1;
        }
        ctl[5] = k;  // tokens found in this window (flushed by all threads)
      }
      __syncthreads();
      {  // flush this window's token positions to global (coalesced)
        const uint32_t k = ctl[5];
        const uint32_t nb = ctl[6];
        for (uint32_t i = t; i < k; i += nt)
          if (nb + i < cap_seq) sc.tokpos[nb + i] = tbuf[i];
        __syncthreads();
        if (t == 0) {
          ctl[6] = nb + k;
          ctl[5] = 0;
        }
      }
    }
    if (t == 0) {
      nseq = ctl[6];
      sc.entry[nch] = pos;
      ctl[0] = (err || !done) ? 1u : 0u;  // no last sequence → truncated stream
      ctl[1] = nseq;
      ctl[3] = nseq > cap_seq ? 1u : 0u;  // scratch too small: caller falls back
    }
    __syncthreads();
  }
  if (ctl[0]) return kCorruptPage;
  PCP_T(2)
  if (ctl[3]) return -1;
  // ---- phase 3: all sequences in parallel: output positions (block scans),
  // literal copies, match records; reference bounds checks ------------------
  {
    const uint32_t S = ctl[1];
    uint32_t* wsum = ctl + 8;
    uint64_t carry = 0;
    for (uint32_t s0 = 0; s0 < S; s0 += nt) {
      const uint32_t i = s0 + t;
      Seq sq{};
      uint32_t len = 0;
      if (i < S) {
        parse_seq(src, n, sc.tokpos[i], sq);  // verified by the skim
        len = sq.lit_len + sq.match_len;
      }
      // block exclusive scan of len
      uint32_t x = len;
      const uint32_t lane = t & 31, w = t >> 5;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if ((int)lane >= o) x += y;
      }
      if (lane == 31) wsum[w] = x;
      __syncthreads();
      uint64_t b0 = carry, tot = 0;
      for (uint32_t k = 0; k < (nt >> 5); ++k) {
        if (k < w) b0 += wsum[k];
        tot += wsum[k];
      }
      const uint64_t op = b0 + x - len;
      // tile tables for the cooperative literal copy (reuse the jump tables)
      uint32_t* t_op = ctl + 72;
      uint32_t* t_src = t_op + nt;
      uint32_t* t_lp = t_src + nt;  // exclusive prefix of literal lengths
      uint32_t lit = (i < S && op + len <= raw_len) ? sq.lit_len : 0u;
      {
        uint32_t y = lit;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
          if ((int)lane >= o) y += z;
        }
        __syncthreads();
        if (lane == 31) wsum[32 + w] = y;
        __syncthreads();
        uint32_t lb = 0, lt = 0;
        for (uint32_t k = 0; k < (nt >> 5); ++k) {
          if (k < w) lb += wsum[32 + k];
          lt += wsum[32 + k];
        }
        t_op[t] = (uint32_t)op;
        t_src[t] = sq.lit_src;
        t_lp[t] = lb + y - lit;
        if (t == 0) ctl[7] = lt;
      }
      __syncthreads();
      {
        const uint32_t L = ctl[7];
        const uint32_t ns = min(nt, S - s0);
        for (uint32_t b = t; b < L; b += nt) {
          uint32_t lo = 0, hi = ns;  // last sequence with t_lp <= b
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (t_lp[mid] <= b) lo = mid;
            else hi = mid;
          }
          const uint32_t k = b - t_lp[lo];
          dst[t_op[lo] + k] = src[t_src[lo] + k];
        }
      }
      if (i < S) {
        if (op + len > raw_len) {
          atomicOr(ctl, 1u);  // literal/match overrun (:137,:150)
        } else {
          if (!sq.last) {
            const uint64_t mo = op + sq.lit_len;
            if (sq.offset > mo) atomicOr(ctl, 1u);  // bad offset (:148)
            sc.m_mo[i] = (uint32_t)mo;
            sc.m_ml[i] = sq.match_len;
            sc.m_off[i] = (uint16_t)sq.offset;
          }
        }
      }
      carry += tot;
      __syncthreads();
    }
    if (t == 0) {
      if (carry != raw_len) ctl[0] = 1u;  // size mismatch (:142)
      ctl[1] = S ? S - 1 : 0;            // matches = every sequence but the last
    }
    __syncthreads();
  }
  if (ctl[0]) return kCorruptPage;
  PCP_T(3)
  // ---- phase 4: matches, in order, by warp 0 through a shared-memory ring --
  // Match dependency chains on these pages are thousands deep (DESIGN.md
  // §4.2), so matches are resolved in stream order by one warp; the other
  // warps of the SM belong to other pages' CTAs.  The ring holds output
  // bytes [hi - kRing, hi); chunks are pulled in from global (literals are
  // final after phase 3) ahead of the match being resolved; sources older
  // than the ring are read back from global (already final).
  const uint32_t M = ctl[1];
  if (t < 32) {
    uint32_t hi = 0, fl = 0;  // ring holds [hi - kRing, hi); global final below fl
    auto move_chunk = [&](uint32_t from, uint32_t end, bool to_ring) {
      if (end - from == kRingChunk && ((uintptr_t)(dst + from) & 15u) == 0) {
        uint4* g4 = reinterpret_cast<uint4*>(dst + from);
        uint4* r4 = reinterpret_cast<uint4*>(ring + (from & (kRing - 1)));
        uint4 v[kRingChunk / 512];
#pragma unroll
        for (int u = 0; u < (int)(kRingChunk / 512); ++u) v[u] = to_ring ? g4[u * 32 + t] : r4[u * 32 + t];
#pragma unroll
        for (int u = 0; u < (int)(kRingChunk / 512); ++u) {
          if (to_ring) r4[u * 32 + t] = v[u];
          else g4[u * 32 + t] = v[u];
        }
      } else {
        for (uint32_t i = from + t; i < end; i += 32) {
          if (to_ring) ring[i & (kRing - 1)] = dst[i];
          else dst[i] = ring[i & (kRing - 1)];
        }
      }
    };
    for (uint32_t base = 0; base < M; base += 32) {
      const uint32_t q = base + t;
      uint32_t r_mo = 0, r_ml = 0, r_off = 1;
      if (q < M) {
        r_mo = sc.m_mo[q];
        r_ml = sc.m_ml[q];
        r_off = sc.m_off[q];
      }
      const uint32_t cnt = min(32u, M - base);
      // ---- group fast path: one match per lane, in dependency waves -------
      {
        const uint32_t g_lo = __shfl_sync(0xffffffffu, r_mo - r_off, 0);  // lowest source start (approx)
        const uint32_t g_end = __shfl_sync(0xffffffffu, r_mo + r_ml, cnt - 1);
        const uint32_t g_first = __shfl_sync(0xffffffffu, r_mo, 0);
        // ensure ring holds [.., g_end): flush final chunks, refill
        bool moved = false;
        while (fl + kRingChunk <= g_first && fl + kRingChunk <= hi) {
          move_chunk(fl, fl + kRingChunk, false);
          fl += kRingChunk;
          moved = true;
        }
        const bool span_ok = g_end - g_first + kRingChunk * 3 <= kRing;
        if (span_ok) {
          while (hi < g_end) {
            const uint32_t end = min(hi + kRingChunk, raw_len);
            while (fl + kRing < end) {
              move_chunk(fl, fl + kRingChunk, false);
              fl += kRingChunk;
            }
            __syncwarp();
            move_chunk(hi, end, true);
            hi = end;
            moved = true;
          }
        }
        if (moved) __syncwarp();
        (void)g_lo;
        const uint32_t lo = hi > kRing ? hi - kRing : 0u;
        const bool act = t < cnt;
        const uint32_t a = r_mo - r_off;
        // every lane's source must be in the ring for the fast path
        const bool src_ok = !act || (a >= lo && r_mo + r_ml <= hi);
        if (span_ok && __all_sync(0xffffffffu, src_ok)) {
          const uint32_t ext_end = min(r_mo, a + r_ml);  // bytes read from earlier output
          uint32_t dep = 0;
#pragma unroll
          for (int d = 1; d < 32; ++d) {
            const uint32_t omo = __shfl_up_sync(0xffffffffu, r_mo, d);
            const uint32_t oml = __shfl_up_sync(0xffffffffu, r_ml, d);
            if ((int)t >= d && act && omo < ext_end && omo + oml > a) dep |= 1u << (t - d);
          }
          uint32_t done = __ballot_sync(0xffffffffu, !act);
          while (done != 0xffffffffu) {
            const bool ready = !((done >> t) & 1u) && (dep & ~done) == 0;
            if (ready) {
              uint8_t* R = ring;
              if (r_off >= r_ml) {  // no self-overlap: loads first, then stores
                uint32_t k = 0;
                for (; k + 4 <= r_ml; k += 4) {
                  const uint8_t b0 = R[(a + k) & (kRing - 1)], b1 = R[(a + k + 1) & (kRing - 1)];
                  const uint8_t b2 = R[(a + k + 2) & (kRing - 1)], b3 = R[(a + k + 3) & (kRing - 1)];
                  R[(r_mo + k) & (kRing - 1)] = b0;
                  R[(r_mo + k + 1) & (kRing - 1)] = b1;
                  R[(r_mo + k + 2) & (kRing - 1)] = b2;
                  R[(r_mo + k + 3) & (kRing - 1)] = b3;
                }
                for (; k < r_ml; ++k) R[(r_mo + k) & (kRing - 1)] = R[(a + k) & (kRing - 1)];
              } else {  // overlapping: the reference's byte-wise forward copy
                for (uint32_t k = 0; k < r_ml; ++k)
                  R[(r_mo + k) & (kRing - 1)] = R[(a + k) & (kRing - 1)];
              }
            }
            __syncwarp();
            done |= __ballot_sync(0xffffffffu, ready);
          }
          if (tm && t == 0) tm[5] += 1;
          continue;
        }
      }
      if (tm && t == 0) tm[6] += 1;
      // ---- slow path: the group one match at a time ------------------------
      for (uint32_t j = 0; j < cnt; ++j) {
        const uint32_t mo = __shfl_sync(0xffffffffu, r_mo, j);
        const uint32_t ml = __shfl_sync(0xffffffffu, r_ml, j);
        const uint32_t off = __shfl_sync(0xffffffffu, r_off, j);
        const uint32_t a = mo - off;
        if (ml <= 32 && mo + ml <= hi && fl + kRingChunk > mo && a + kRing >= hi) {
          // fast path: no ring traffic, one pass, source inside the ring
          uint32_t r = t - off * __float2uint_rz(__fdividef((float)t + 0.5f, (float)off));
          r = off >= ml ? t : r;
          const uint8_t v = ring[(a + r) & (kRing - 1)];
          if (t < ml) ring[(mo + t) & (kRing - 1)] = v;
          __syncwarp();
          continue;
        }
        bool moved = false;
        while (fl + kRingChunk <= mo && fl + kRingChunk <= hi) {  // final: write back
          move_chunk(fl, fl + kRingChunk, false);
          fl += kRingChunk;
          moved = true;
        }
        while (hi < mo + ml) {  // pull the next chunk (literals final) into the ring
          const uint32_t end = min(hi + kRingChunk, raw_len);
          // the slots about to be reused hold bytes < mo (final): write back first
          while (fl + kRing < end) {
            move_chunk(fl, fl + kRingChunk, false);
            fl += kRingChunk;
          }
          __syncwarp();
          move_chunk(hi, end, true);
          hi = end;
          moved = true;
        }
        if (moved) __syncwarp();
        const uint32_t lo = hi > kRing ? hi - kRing : 0u;
        if (ml <= 32 && a >= lo) {  // common case: one pass, source in the ring
          if (t < ml) {
            uint32_t r = t;
            if (off < ml) {  // periodic copy: r = t mod off (t < 32, exact in float)
              r = t - off * __float2uint_rz(__fdividef((float)t + 0.5f, (float)off));
            }
            ring[(mo + t) & (kRing - 1)] = ring[(a + r) & (kRing - 1)];
          }
        } else {
          for (uint32_t i = t; i < ml; i += 32) {
            const uint32_t r = off >= ml ? i : i % off;
            const uint32_t sp = a + r;
            const uint8_t v = sp >= lo ? ring[sp & (kRing - 1)] : dst[sp];
            ring[(mo + i) & (kRing - 1)] = v;
          }
        }
        __syncwarp();
      }
    }
    if (M) {
      while (fl < hi) {
        const uint32_t end = min(fl + kRingChunk, hi);
        move_chunk(fl, end, false);
        fl = end;
      }
    }
  }
  __syncthreads();
  PCP_T(4)
#undef PCP_T
  return kOk;
}

}  // namespace lz4p
}  // namespace pcp
