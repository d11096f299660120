// lz4_parallel.cuh — CTA-parallel decode of ONE LZ4 block (the reference
// writes one block per page, lz4_block.cpp:33-110), output byte-identical to
// lz4::decompress (lz4_block.cpp:113-156) with the same error verdicts.
//
// The token chain of an LZ4 block is serial; on the reference's quantised
// pages it is ~1 sequence per 8 B (avg literal ~4 B, match ~4 B; SURVEY.md
// App. A).  Speculative parsing from chunk starts was measured and rejected
// (most chunks never re-synchronise).  The decoder instead:
//
//  1-2. skim (k_page_decode): 2 KB windows of the payload are staged in
//     shared memory by cp.async.bulk (TMA, one mbarrier per buffer) a window
//     ahead.  Warps 1-7 fill window w+1's jump table d(p) = distance to the
//     next token if one started at p (plus two- and four-token jumps) while
//     one lane of the last warp walks window w with one round of two
//     independent shared loads per one, two or four tokens, storing a u32
//     step record per step; the fill warps expand the records into global
//     token positions.  Windows inside long literals are skipped.
//  3. all sequences in parallel: block scans give output positions; literals
//     are copied in 16-B aligned output chunks; match records are emitted
//     with every reference bounds check (all violations are kCorruptPage, so
//     verdicts do not depend on order).
//  4. matches (k_page_matches): resolved in stream order through a 16 KB
//     shared-memory ring of the output.  Runs of matches whose output span
//     fits 2 KB are resolved by pointer jumping (every byte points at its
//     source, doubling until it reaches a final byte, then one gather); the
//     rest go one match per lane in dependency waves.  Overlapping copies use
//     dst[mo+i] = dst[mo-off + i % off], the closed form of the byte-wise copy.
#pragma once

#include <cstdint>

#include "device_util.cuh"
#include "pcp_internal.h"

namespace pcp {
namespace lz4p {

constexpr uint32_t kChunk = 2048;      // compressed bytes per skim window / parse chunk
constexpr uint32_t kRing = 16384;      // shared-memory output window (bytes)
constexpr uint32_t kStageTail = 128;   // staged bytes past a window for its last tokens
constexpr uint32_t kStageBytes = kChunk + kStageTail + 32;  // + 16-B alignment slack (TMA)
// ctl[0..72) control; jump tables d|d2 [2][kChunk] u32; stage buffers; d4
// tables [2][kChunk] u16; walker step records [2][kChunk] u32
constexpr uint32_t kSmemWords = 72 + 2 * kChunk + (2 * kStageBytes) / 4 + kChunk + 2 * kChunk;
constexpr uint32_t kRingChunk = 4096;  // refill granule
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kDoubleSpan = 2048;  // group output span resolved by pointer jumping

// Per-page scratch layout (host computes the size with scratch_bytes()).
__host__ __device__ inline uint32_t n_chunks(uint64_t pay) {
  return (uint32_t)((pay + kChunk - 1) / kChunk);
}
__host__ __device__ inline uint64_t match_capacity(uint64_t pay) { return pay / 6 + 64; }

__host__ __device__ inline uint64_t scratch_bytes(uint64_t pay) {
  return 64 + match_capacity(pay) * 16 + 256;
}

// Per-page scratch: a header (phase-4 hand-off between k_page_decode and
// k_page_matches), match records and the token positions of the skim.
struct Scratch {
  uint32_t* hdr;       // [0] matches M, [1] 1 = phase 4 pending
  uint32_t* m_mo;      // match output start
  uint32_t* m_ml;      // match length
  uint16_t* m_off;     // offset
  uint32_t* tokpos;    // true token positions, in stream order
};

__device__ inline Scratch carve_scratch(uint8_t* p, uint64_t pay) {
  Scratch s;
  s.hdr = reinterpret_cast<uint32_t*>(p);
  uint32_t* m = s.hdr + 16;
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

// LZ4 length extension (lz4_block.cpp:123-129 / :143-149): acc += bytes
// until the first byte != 255 (inclusive) or acc reaches 0x7fffffff; false
// if the stream ends first.  Raw-float pages carry literal runs of megabytes
// whose length field is thousands of 255 bytes, so 16-B aligned stretches
// are scanned 128 bytes per step with eight independent loads; the guard
// and the truncation point are exactly the byte loop's.
__device__ __forceinline__ bool ext_len(const uint8_t* __restrict__ src, uint32_t n, uint32_t& ip,
                                        uint32_t& acc) {
  while (true) {
    if (ip >= n) return false;
    // the 128-B block of 16-B aligned words starting at or below ip (reads
    // <= 15 bytes before ip, inside the page header / payload)
    const uint32_t sh = (uint32_t)((reinterpret_cast<uintptr_t>(src) + ip) & 15u);
    if (ip + 128 - sh <= n && acc < 0x7fffffffu - 255u * 128u) {
      const uint4* q = reinterpret_cast<const uint4*>(src + ip - sh);
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = q[u];
      uint32_t j = 128;  // first byte != 255 at or after offset sh
#pragma unroll
      for (int u = 7; u >= 0; --u) {
        const uint32_t w4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int e = 3; e >= 0; --e) {
          uint32_t x = ~w4[e];  // nonzero bytes = bytes != 255
          const int b0 = 16 * u + 4 * e;
          if (b0 + 4 <= (int)sh) x = 0;  // word entirely before ip
          else if (b0 < (int)sh) x &= 0xFFFFFFFFu << (8 * (sh - b0));
          if (x) j = b0 + (__ffs(x) - 1) / 8;
        }
      }
      if (j == 128) {
        acc += 255u * (128u - sh);
        ip += 128u - sh;
        continue;
      }
      acc += 255u * (j - sh) + src[ip - sh + j];
      ip += j - sh + 1;
      return true;
    }
    const uint32_t b = src[ip++];
    acc += b;
    if (b != 255 || acc >= 0x7fffffffu) return true;
  }
}

__device__ __forceinline__ bool parse_seq(const uint8_t* __restrict__ src, uint32_t n, uint32_t ip,
                                          Seq& s) {
  if (ip >= n) return false;
  const uint32_t token = src[ip++];
  uint32_t lit = token >> 4;
  if (lit == 15 && !ext_len(src, n, ip, lit)) return false;
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
  if (ml == 15 && !ext_len(src, n, ip, ml)) return false;
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

// parse_seq over a staged window (bytes [c0, se) in shared memory) without
// touching global memory: 0 malformed, 1 parsed, 2 needs a byte in [se, n)
// (the walker then parses that position from global).  Checks in
// parse_seq's order, so verdicts 0/1 are parse_seq's.
__device__ __forceinline__ int parse_seq_win(const uint8_t* buf, uint32_t c0, uint32_t se,
                                             uint32_t n, uint32_t ip, Seq& s) {
  if (ip >= n) return 0;
  if (ip >= se) return 2;
  const uint32_t token = buf[ip++ - c0];
  uint32_t lit = token >> 4;
  if (lit == 15) {
    uint32_t b;
    do {
      if (ip >= n) return 0;
      if (ip >= se) return 2;
      b = buf[ip++ - c0];
      lit += b;
    } while (b == 255 && lit < 0x7fffffffu);
  }
  if ((uint64_t)ip + lit > n) return 0;
  s.lit_src = ip;
  s.lit_len = lit;
  ip += lit;
  if (ip == n) {
    s.last = true;
    s.match_len = 0;
    s.offset = 0;
    s.next = n;
    return 1;
  }
  if (ip + 2 > n) return 0;
  if (ip + 2 > se) return 2;
  s.offset = (uint32_t)buf[ip - c0] | ((uint32_t)buf[ip + 1 - c0] << 8);
  ip += 2;
  if (s.offset == 0) return 0;
  uint32_t ml = token & 15;
  if (ml == 15) {
    uint32_t b;
    do {
      if (ip >= n) return 0;
      if (ip >= se) return 2;
      b = buf[ip++ - c0];
      ml += b;
    } while (b == 255 && ml < 0x7fffffffu);
  }
  s.match_len = ml + 4;
  s.last = false;
  s.next = ip;
  return 1;
}

// Barrier among the fill warps only (warps 1..), id 1.
__device__ __forceinline__ void named_sync_fill(uint32_t nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
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

// Phases 1-3 of one page with the whole CTA (`ctl`: kSmemWords of shared
// memory).  Returns the status (same on all threads): kOk with ctl[1] =
// matches left for phase 4, kCorruptPage, or -1 (scratch too small: the
// caller falls back to the warp decoder).
__device__ inline int32_t decode_prefix(const uint8_t* __restrict__ src, uint32_t n,
                                        uint8_t* __restrict__ dst, uint32_t raw_len, Scratch sc,
                                        uint32_t* ctl, long long* tm = nullptr) {
#define PCP_T(i) \
  if (tm && threadIdx.x == 0) tm[i] = clock64();
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  const uint32_t nch = n_chunks(n);

  if (t == 0) ctl[0] = 0;            // error
  if (n == 0) return kCorruptPage;   // "truncated stream" (:134)
  PCP_T(0)
  // ---- phases 1+2: skim the token chain ------------------------------------
  // Window w = compressed bytes [w*kChunk, (w+1)*kChunk).  Warps 1.. fill the
  // jump table of window w+1 — d[p] = distance from p to the next token if a
  // token started at p (bit 31: malformed, bit 30: last sequence, bit 29:
  // header runs past the staged bytes) — while warp 0's lane 0 walks the
  // true chain through window w with one shared-memory lookup per sequence,
  // writing each token position straight to global.  Window bytes arrive by
  // TMA bulk copy one window ahead (mbarrier per buffer), so neither side
  // waits on HBM.
  {
    // per window buffer b: jt[b][kChunk] u32 = d (low 16 bits) | d2 << 16
    uint32_t* jt = ctl + 72;
    uint8_t* wb = reinterpret_cast<uint8_t*>(ctl + 72 + 2 * kChunk);  // 2 x kStageBytes bytes
    // four-token jumps d4 = d2(p) + d2(p + d2(p)) (u16, 0 = none): [2][kChunk]
    uint16_t* j4 = reinterpret_cast<uint16_t*>(ctl + 72 + 2 * kChunk + (2 * kStageBytes) / 4);
    // walker step records [2][kChunk] (u32): lp | code << 11 | k << 13 per
    // step of 1 (code 0), 2 (1) or 4 (2) tokens starting at window offset lp,
    // k = the step's first token within the window.  The fill warps expand
    // them from the window's jump table into sc.tokpos after the next
    // barrier: one shared store per step keeps the lone walker's MIO queue
    // short (it used to store every position and load the fourth token's hop)
    uint32_t* tw = reinterpret_cast<uint32_t*>(j4 + 2 * kChunk);
    uint64_t* sbar = reinterpret_cast<uint64_t*>(ctl + 64);     // stage barriers (ctl[64..67])
    const uintptr_t sbase = reinterpret_cast<uintptr_t>(src);
    // window w's bytes [c0, min(c0 + kChunk + kStageTail, n)) as the 16-B
    // aligned superset; readers index buf0 + ((src + c0) & 15)
    // ctl[56 + b] = window staged in buffer b (~0u: none), ctl[58 + b] = stagings
    // issued into buffer b (its mbarrier's phase parity is (count - 1) & 1)
    auto stage_async = [&](uint32_t w) {  // one thread
      const uint32_t b = w & 1u;
      ctl[56 + b] = w;
      ctl[58 + b] += 1;
      const uint32_t e = min(w * kChunk + kChunk + kStageTail, n);
      const uintptr_t g0 = (sbase + w * kChunk) & ~uintptr_t(15);
      const uintptr_t g1 = (sbase + e + 15) & ~uintptr_t(15);
      const uint32_t bytes = (uint32_t)(g1 - g0);
      dev::mbar_expect_tx(&sbar[b], bytes);
      dev::bulk_g2s(wb + b * kStageBytes, reinterpret_cast<const void*>(g0), bytes, &sbar[b]);
    };
    // jump-table fill: the common header (every byte inside the staged
    // window, no 255-continued length) in two levels of independent
    // shared-memory loads; anything else goes through parse_seq_win.
    auto fill = [&](uint32_t w, uint32_t* tab32, uint32_t tid, uint32_t nthr) {
      uint16_t* tab = reinterpret_cast<uint16_t*>(tab32);  // low halves: tab[2 * lp]
      const uint32_t c0 = w * kChunk, c1 = min(c0 + kChunk, n);
      const uint8_t* buf = wb + (w & 1u) * kStageBytes + ((sbase + c0) & 15u);
      const uint32_t se = min(c0 + kChunk + kStageTail, n);
      for (uint32_t p = c0 + tid; p < c1; p += nthr) {
        const uint32_t lp = p - c0;
        const uint32_t tok = buf[lp];
        const uint32_t e1 = p + 1 < se ? buf[lp + 1] : 255u;
        uint32_t lit = tok >> 4, hdr = 1;
        if (lit == 15) {
          lit += e1;
          hdr = 2;
        }
        const uint32_t ip = p + hdr + lit;  // offset position (if not the last sequence)
        uint32_t v = 0;
        bool general = !(!(tok >= 0xF0u && e1 == 255u) && ip + 3 <= se && ip + 3 <= n);
        if (!general) {
          const uint32_t o = ip - c0;
          const uint32_t off = (uint32_t)buf[o] | ((uint32_t)buf[o + 1] << 8);
          const bool ml15 = (tok & 15u) == 15u;
          if (ml15 && buf[o + 2] == 255u) general = true;  // long match-length run
          else v = off == 0 ? 0x80000000u : (ip + 2 + (ml15 ? 1u : 0u)) - p;
        }
        if (general) {
          Seq sq;
          const int r = parse_seq_win(buf, c0, se, n, p, sq);
          v = r == 0 ? 0x80000000u : r == 2 ? 0x20000000u : sq.last ? 0x40000000u : sq.next - p;
        }
        // u16 entry: distance, or 0xFFFF = walker parses this position from
        // global (malformed / last / past the stage / distance >= 0xFFFF)
        tab[2 * lp] = (v & 0xE0000000u) || v >= 0xFFFFu ? (uint16_t)0xFFFFu : (uint16_t)v;
      }
    };
    // two-token jumps: d2[p] = d[p] + d[p + d[p]] when both hops are plain
    // and the second token starts in this window, else 0
    auto fill2 = [&](uint32_t w, uint32_t* tab32, uint32_t tid, uint32_t nthr) {
      const uint16_t* tab = reinterpret_cast<const uint16_t*>(tab32);
      uint16_t* tab2 = reinterpret_cast<uint16_t*>(tab32) + 1;  // high halves
      const uint32_t c0 = w * kChunk, len = min(c0 + kChunk, n) - c0;
      for (uint32_t lp = tid; lp < len; lp += nthr) {
        const uint32_t a = tab[2 * lp];
        uint32_t r = 0;
        if (a != 0xFFFFu && lp + a < len) {
          const uint32_t b = tab[2 * (lp + a)];
          if (b != 0xFFFFu && a + b < 0xFFFFu) r = a + b;
        }
        tab2[2 * lp] = (uint16_t)r;
      }
    };
    auto fill4 = [&](uint32_t w, const uint32_t* tab32, uint16_t* t4, uint32_t tid, uint32_t nthr) {
      const uint32_t c0 = w * kChunk, len = min(c0 + kChunk, n) - c0;
      for (uint32_t lp = tid; lp < len; lp += nthr) {
        const uint32_t b = tab32[lp] >> 16;
        uint32_t r = 0;
        if (b && lp + b < len) {
          const uint32_t b2 = tab32[lp + b] >> 16;
          if (b2 && b + b2 < 0xFFFFu) r = b + b2;
        }
        t4[lp] = (uint16_t)r;
      }
    };
    // window w's step records -> token positions in sc.tokpos[base ..)
    // (reads window w's jump table, still intact: it is refilled for window
    // w+2 only after the caller's barrier)
    const uint32_t cap_seq = (uint32_t)match_capacity(n);
    auto expand = [&](uint32_t w, uint32_t cnt, uint32_t base, uint32_t tid, uint32_t nthr) {
      const uint32_t* tab = jt + (w & 1u) * kChunk;
      const uint32_t* rec = tw + (w & 1u) * kChunk;
      const uint32_t c0 = w * kChunk;
      for (uint32_t i = tid; i < cnt; i += nthr) {
        const uint32_t e = rec[i];
        const uint32_t lp = e & 0x7FFu, code = (e >> 11) & 3u, o = base + (e >> 13);
        if (o < cap_seq) sc.tokpos[o] = c0 + lp;
        if (code) {
          const uint32_t x = tab[lp];
          if (o + 1 < cap_seq) sc.tokpos[o + 1] = c0 + lp + (x & 0xFFFFu);
          if (code == 2) {
            const uint32_t b = x >> 16;
            if (o + 2 < cap_seq) sc.tokpos[o + 2] = c0 + lp + b;
            if (o + 3 < cap_seq) sc.tokpos[o + 3] = c0 + lp + b + (tab[lp + b] & 0xFFFFu);
          }
        }
      }
    };
    if (t == 0) {
      dev::mbar_init(&sbar[0], 1);
      dev::mbar_init(&sbar[1], 1);
      dev::fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
      ctl[58] = ctl[59] = 0;
      ctl[57] = ~0u;
      stage_async(0);
      if (nch > 1) stage_async(1);
      ctl[54] = 0;  // walker position at the start of window w: ctl[54 + (w & 1)]
    }
    dev::mbar_wait(&sbar[0], 0);
    fill(0, jt, t, nt);
    __syncthreads();
    fill2(0, jt, t, nt);
    __syncthreads();
    fill4(0, jt, j4, t, nt);
    __syncthreads();
    long long a_walk = 0, a_fill = 0;  // PCP_LZ4_TIMING
    // the walker is lane 0 of the LAST warp: the SMSP arbiter issues the
    // highest warp id first, and the walker's serial chain is the skim's
    // critical path; warps 0 .. nw-2 fill tables
    const uint32_t wk = nt - 32;  // walker thread; fill threads are t < wk
    uint32_t pos = 0;  // walker state
    uint32_t err = 0, done = 0, nseq = 0;
    for (uint32_t w = 0; w < nch; ++w) {
      if (t < wk) {
        const long long f0 = (tm && t == 0) ? clock64() : 0;
        if (w > 0) {  // window w-1's token positions -> global
          const uint32_t pb = (w - 1) & 1u;
          expand(w - 1, ctl[50 + pb], ctl[52 + pb], t, wk);
          named_sync_fill(wk);  // its jump table is refilled (window w+1) below
        }
        // window w's buffer was last read by fill(w) before the previous
        // barrier: refill it with window w+2 (async), then fill window w+1
        // a window the walker has already passed (inside a long literal, or
        // after the last sequence) is never read: skip its tables, and do not
        // even stage it when that is known an iteration ahead (a C2 page is
        // two-thirds such windows; staging them put one TMA latency per
        // window on the critical path).  Uniform across the fill warps: the
        // walker publishes the next window's start position in the other
        // parity slot, and the stager records what each buffer holds.
        const uint32_t wpos = ctl[54 + (w & 1u)];
        if (t == 0) {
          if (w + 2 < nch && wpos < (w + 3) * kChunk) {
            dev::fence_proxy_async();
            stage_async(w + 2);
          } else {
            ctl[56 + (w & 1u)] = ~0u;
          }
        }
        const bool need = wpos < (w + 2) * kChunk;
        const uint32_t b1 = (w + 1) & 1u;
        if (w + 1 < nch && ctl[56 + b1] == w + 1) dev::mbar_wait(&sbar[b1], (ctl[58 + b1] - 1) & 1u);
        if (w + 1 < nch && need) {
          uint32_t* tb = jt + ((w + 1) & 1u) * kChunk;
          fill(w + 1, tb, t, wk);
          named_sync_fill(wk);
          fill2(w + 1, tb, t, wk);
          named_sync_fill(wk);
          fill4(w + 1, tb, j4 + ((w + 1) & 1u) * kChunk, t, wk);
        }
        if (tm && t == 0) a_fill += clock64() - f0;
      } else if (t == wk) {
        const long long w0 = tm ? clock64() : 0;
        const uint32_t* tab = jt + (w & 1u) * kChunk;
        const uint16_t* t4 = j4 + (w & 1u) * kChunk;
        const uint32_t c0 = w * kChunk, len = min(c0 + kChunk, n) - c0;
        uint32_t* tr = tw + (w & 1u) * kChunk;
        uint32_t k = 0, r = 0;  // tokens / step records of this window (all start inside it)
        if (!done && pos < c0 + len) {
          uint32_t lp = pos - c0;
          while (true) {
            // hot loop: one round of two independent LDS (d|d2 and d4 at
            // lp) per one, two or four tokens, branch-free step selection
            uint32_t x = tab[lp], f = t4[lp];  // f: four-token jump (0: none)
            while ((x & 0xFFFFu) != 0xFFFFu) {
              const uint32_t a = x & 0xFFFFu, b = x >> 16;
              const uint32_t code = f ? 2u : (b ? 1u : 0u);
              tr[r++] = lp | (code << 11) | (k << 13);
              k += 1u << code;
              lp += f ? f : (b ? b : a);
              if (lp >= len) break;
              x = tab[lp];
              f = t4[lp];
            }
            if (lp >= len) break;
            // entry 0xFFFF: parse this position exactly from global
            tr[r++] = lp | (k << 13);
            ++k;
            Seq sq;
            if (!parse_seq(src, n, c0 + lp, sq)) {
              err = done = 1;
              break;
            }
            if (sq.last) {
              done = 1;
              break;
            }
            lp = sq.next - c0;
            if (lp >= len) break;
          }
          pos = done ? n : c0 + lp;
        }
        ctl[50 + (w & 1u)] = r;
        ctl[52 + (w & 1u)] = nseq;
        nseq += k;
        ctl[54 + ((w + 1) & 1u)] = pos;  // read by the fill warps in iteration w+1
        if (tm) a_walk += clock64() - w0;
      }
      __syncthreads();
    }
    {  // the last window's token positions -> global
      const uint32_t pb = (nch - 1) & 1u;
      expand(nch - 1, ctl[50 + pb], ctl[52 + pb], t, nt);
    }
    if (tm && t == wk) tm[8] = a_walk;
    if (tm && t == 0) tm[9] = a_fill;
    if (t == wk) {
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
      // tile tables for the cooperative literal copy (reuse the jump tables):
      // each literal is cut into 16-B aligned output chunks; a chunk prefix
      // over the tile maps thread work items to (sequence, chunk)
      uint32_t* t_op = ctl + 72;
      uint32_t* t_src = t_op + nt;
      uint32_t* t_len = t_src + nt;
      uint32_t* t_cp = t_len + nt;  // exclusive prefix of chunk counts
      const uint32_t lit = (i < S && op + len <= raw_len) ? sq.lit_len : 0u;
      // chunk boundaries on absolute addresses (dst may be unaligned)
      const uint32_t doff = (uint32_t)(reinterpret_cast<uintptr_t>(dst) & 15u);
      const uint32_t nck = lit ? (uint32_t)((op + doff + lit + 15) / 16 - (op + doff) / 16) : 0u;
      {
        uint32_t y = nck;
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
        t_len[t] = lit;
        t_cp[t] = lb + y - nck;
        if (t == 0) ctl[7] = lt;
      }
      __syncthreads();
      {
        const uint32_t C = ctl[7];
        const uint32_t ns = min(nt, S - s0);
        for (uint32_t c = t; c < C; c += nt) {
          uint32_t lo = 0, hi = ns;  // last sequence with t_cp <= c
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (t_cp[mid] <= c) lo = mid;
            else hi = mid;
          }
          const uint32_t d = t_op[lo], L = t_len[lo];
          // this chunk's aligned start, in dst + doff coordinates
          const uint32_t a0 = ((d + doff) / 16 + (c - t_cp[lo])) * 16;
          const uint32_t b0 = max(a0, d + doff) - doff, b1 = min(a0 + 16, d + doff + L) - doff;
          const uint8_t* sp = src + t_src[lo] + (b0 - d);
          if (b1 - b0 == 16) {  // full chunk: one aligned 16-B store at dst + b0
            const uintptr_t sa = reinterpret_cast<uintptr_t>(sp);
            const uint32_t sh = (uint32_t)(sa & 3u) * 8u;
            const uint32_t* q = reinterpret_cast<const uint32_t*>(sa & ~uintptr_t(3));
            const uint32_t w0 = q[0], w1 = q[1], w2 = q[2], w3 = q[3];
            uint4 v;
            if (sh) {
              const uint32_t w4 = q[4];  // <= 3 bytes past the literal (payload slack)
              v = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh),
                             __funnelshift_r(w2, w3, sh), __funnelshift_r(w3, w4, sh));
            } else {
              v = make_uint4(w0, w1, w2, w3);
            }
            *reinterpret_cast<uint4*>(dst + b0) = v;
          } else {
            for (uint32_t b = b0; b < b1; ++b) dst[b] = sp[b - b0];
          }
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
#undef PCP_T
  return kOk;
}

// Named barrier 2 over the phase-4 warps; the OR of `v` over them.
__device__ __forceinline__ void bar_jump(uint32_t nthreads) {
  asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ bool bar_jump_or(uint32_t nthreads, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, 2, %2, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(nthreads)
      : "memory");
  return r != 0;
}

// Byte-level pointer jumping over the output span [g0, g0 + L) by threads
// tid < nthr (nthr = 32: warp 0 alone; more: warp 0 + helper warps, synced
// by named barrier 2): src(b) = b - off inside a match (the forward copy's
// semantics, self-overlap included), b for literals; bytes below the span are
// final in the ring.  Doubling until every pointer reaches a final byte takes
// log2(chain depth) rounds instead of one dependency wave per link.  On entry
// pidx holds the pointers; on exit the span's bytes are final in the ring.
__device__ __forceinline__ void jump_rounds(uint8_t* ring, uint32_t* pidx, uint32_t g0, uint32_t L,
                                            uint32_t tid, uint32_t nthr) {
  for (int round = 0; round < 16; ++round) {  // depth <= L <= 2^11
    bool ch = false;
    for (uint32_t b0 = tid; b0 < L; b0 += 4 * nthr) {  // 4 bytes per thread in flight
      uint32_t p[4], q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t b = b0 + nthr * u;
        p[u] = b < L ? pidx[b] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = (b0 + nthr * u < L && p[u] >= g0) ? pidx[p[u] - g0] : p[u];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q[u] != p[u]) {
          pidx[b0 + nthr * u] = q[u];
          ch = true;
        }
    }
    if (nthr > 32) {
      if (!bar_jump_or(nthr, ch)) break;
    } else {
      __syncwarp();
      if (!__any_sync(0xffffffffu, ch)) break;
    }
  }
  // every final source is a literal of the span or a byte below it: those
  // never change, so the gather has no read/write hazard
  for (uint32_t b0 = tid; b0 < L; b0 += 4 * nthr) {
    uint32_t p[4];
    uint8_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = b0 + nthr * u < L ? pidx[b0 + nthr * u] : g0 + b0 + nthr * u;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = p[u] != g0 + b0 + nthr * u ? ring[p[u] & (kRing - 1)] : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (p[u] != g0 + b0 + nthr * u) ring[(g0 + b0 + nthr * u) & (kRing - 1)] = v[u];
  }
  if (nthr > 32) bar_jump(nthr);
  else __syncwarp();
}

// Helper warps of phase 4 (threadIdx.x >= 32, nthr = all phase-4 threads):
// wait for warp 0's span command (cmd[0] = 1, g0, L; 0 = page done), take a
// share of the span init and of every jump round, in lockstep with warp 0's
// barriers in decode_matches.
// Match pointers of matches [q0, q0 + cnt) into pidx (span starting at g0),
// one match per thread; records from shared memory (srec: mo[256], ml[256],
// off[256], staged by warp 0) or, without it, from the scratch.
__device__ __forceinline__ void span_pointers(const Scratch& sc, const uint32_t* srec, uint32_t* pidx,
                                              uint32_t g0, uint32_t q0, uint32_t cnt, uint32_t tid,
                                              uint32_t nthr) {
  for (uint32_t i = tid; i < cnt; i += nthr) {
    const uint32_t mo = srec ? srec[i] : sc.m_mo[q0 + i];
    const uint32_t ml = srec ? srec[256 + i] : sc.m_ml[q0 + i];
    const uint32_t a = mo - (srec ? srec[512 + i] : sc.m_off[q0 + i]);
    for (uint32_t j = 0; j < ml; ++j) pidx[mo - g0 + j] = a + j;
  }
}

__device__ inline void matches_helper(const Scratch& sc, uint8_t* ring, uint32_t* pidx,
                                      volatile uint32_t* cmd, uint32_t nthr, const uint32_t* srec) {
  const uint32_t tid = threadIdx.x;
  while (true) {
    bar_jump(nthr);  // B1: command published
    if (cmd[0] == 0) return;
    const uint32_t g0 = cmd[1], L = cmd[2], q0 = cmd[3], cnt = cmd[4];
    for (uint32_t b = tid; b < L; b += nthr) pidx[b] = g0 + b;
    bar_jump(nthr);  // B2: span initialised
    span_pointers(sc, srec, pidx, g0, q0, cnt, tid, nthr);
    bar_jump(nthr);  // B3: match pointers written
    jump_rounds(ring, pidx, g0, L, tid, nthr);
  }
}

// Phase 4 of one page by warp 0 (lane = threadIdx.x & 31): the M matches
// recorded by decode_prefix, in order, through a shared-memory ring (`ring`:
// kRing bytes).  With nthr > 32, warps 1.. run matches_helper and share the
// pointer-jumping spans (cmd: 3 words of shared memory).
__device__ inline void decode_matches(uint8_t* __restrict__ dst, uint32_t raw_len, Scratch sc,
                                      uint32_t M, uint8_t* ring, uint32_t* pidx,
                                      long long* tm = nullptr, uint32_t nthr = 32,
                                      volatile uint32_t* cmd = nullptr, uint32_t* srec = nullptr) {
  const uint32_t t = threadIdx.x & 31u;
  {

    uint32_t hi = 0, fl = 0;  // ring holds [max(hi - kRing, vlo), hi); global final below fl
    uint32_t vlo = 0;         // start of the ring's valid bytes since the last skip
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
    // chunks at or above hi and wholly below the chunk before g_first hold
    // no match output (matches come in output order, and every earlier one
    // landed below hi), so they are final in dst already -- phase 3 wrote the
    // literals there.  Jump over them instead of streaming them through the
    // ring (a C2 page's 24 KB float literals, 64 times) after writing the
    // ring back.  Sources below the new window are read from dst.
    auto skip_final = [&](uint32_t g_first) -> bool {
      const uint32_t c = g_first & ~(kRingChunk - 1u);
      if (c < hi + 2u * kRingChunk) return false;
      while (fl < hi) {
        const uint32_t end = min(fl + kRingChunk, hi);
        move_chunk(fl, end, false);
        fl = end;
      }
      fl = hi = vlo = c - kRingChunk;
      return true;
    };
    // flush final chunks below g_first, refill the ring up to g_end; false if
    // [g_first, g_end) cannot sit in the ring together with its sources
    auto ensure_ring = [&](uint32_t g_first, uint32_t g_end) -> bool {
      bool moved = skip_final(g_first);
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
      return span_ok;
    };
    // byte-level pointer jumping over the output span [g0, g0 + L): src(b) =
    // b - off inside a match (the forward copy's semantics, self-overlap
    // included), b for literals; bytes below the span are final in the ring.
    // Doubling until every pointer reaches a final byte takes log2(chain
    // depth) rounds instead of one dependency wave per link.  The caller
    // fills pidx with the matches' pointers after init_span.
    // span [g0, g0 + L) for pointer jumping (see jump_rounds): publish it to
    // the helper warps, initialise pidx (all phase-4 threads)
    // matches [q0, q0 + cnt) covering the span [g0, g0 + L): init pidx,
    // write the match pointers, jump (all phase-4 threads)
    uint32_t smo[8], sml[8], soff[8];  // this iteration's records (lane t: base + 32k + t)
    auto span_jump = [&](uint32_t g0, uint32_t L, uint32_t q0, uint32_t cnt) {
      if (srec) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          srec[32 * k + t] = smo[k];
          srec[256 + 32 * k + t] = sml[k];
          srec[512 + 32 * k + t] = soff[k];
        }
      }
      if (nthr > 32) {
        if (t == 0) {
          cmd[1] = g0;
          cmd[2] = L;
          cmd[3] = q0;
          cmd[4] = cnt;
          cmd[0] = 1;
        }
        bar_jump(nthr);  // B1
      }
      for (uint32_t b = t; b < L; b += nthr) pidx[b] = g0 + b;
      if (nthr > 32) bar_jump(nthr);  // B2
      else __syncwarp();
      if (!srec) __syncwarp();
      span_pointers(sc, srec, pidx, g0, q0, cnt, t, nthr);
      if (nthr > 32) bar_jump(nthr);  // B3
      else __syncwarp();
      jump_rounds(ring, pidx, g0, L, t, nthr);
    };
    uint32_t step = 32;
    // the next 256 records, loaded an iteration ahead on the guess that this
    // iteration is a full super-group (the usual case in label regions)
    uint32_t pmo[8], pml[8], poff[8], pbase = ~0u;
    auto load_recs = [&](uint32_t b, uint32_t (&mo)[8], uint32_t (&ml)[8], uint32_t (&of)[8]) {
      const uint32_t c = min(256u, M - b);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t q = b + 32 * k + t;
        const bool v = q < b + c;
        mo[k] = v ? sc.m_mo[q] : 0u;
        ml[k] = v ? sc.m_ml[q] : 0u;
        of[k] = v ? sc.m_off[q] : 1u;
      }
    };
    for (uint32_t base = 0; base < M; base += step) {
      step = 32;
      // ---- super-group: up to 8 x 32 consecutive matches in one jump pass
      // when their output span is <= kDoubleSpan (dense label regions)
      const uint32_t cntS = min(256u, M - base);
      if (pbase == base) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          smo[k] = pmo[k];
          sml[k] = pml[k];
          soff[k] = poff[k];
        }
      } else {
        load_recs(base, smo, sml, soff);
      }
      pbase = base + cntS;
      if (pbase < M) load_recs(pbase, pmo, pml, poff);
      if (pidx && cntS > 32) {
        const uint32_t lastk = (cntS - 1) >> 5, lastl = (cntS - 1) & 31u;
        uint32_t e_last = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if ((uint32_t)k == lastk) e_last = smo[k] + sml[k];
        const uint32_t s_end = __shfl_sync(0xffffffffu, e_last, lastl);
        const uint32_t s_first = __shfl_sync(0xffffffffu, smo[0], 0);
        if (s_end - s_first <= kDoubleSpan && ensure_ring(s_first, s_end)) {
          const uint32_t lo = max(hi > kRing ? hi - kRing : 0u, vlo);
          bool ok = true;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (32u * k + t < cntS) ok = ok && smo[k] - soff[k] >= lo && smo[k] + sml[k] <= hi;
          if (__all_sync(0xffffffffu, ok)) {
            span_jump(s_first, s_end - s_first, base, cntS);
            if (tm && t == 0) tm[7] += 1;
            step = cntS;
            continue;
          }
        }
      }
      const uint32_t r_mo = smo[0], r_ml = sml[0], r_off = soff[0];
      const uint32_t cnt = min(32u, M - base);
      // ---- group fast path: one match per lane ----------------------------
      {
        const uint32_t g_end = __shfl_sync(0xffffffffu, r_mo + r_ml, cnt - 1);
        const uint32_t g_first = __shfl_sync(0xffffffffu, r_mo, 0);
        const bool span_ok = ensure_ring(g_first, g_end);
        const uint32_t lo = max(hi > kRing ? hi - kRing : 0u, vlo);
        const bool act = t < cnt;
        const uint32_t a = r_mo - r_off;
        // every lane's source must be in the ring for the fast path
        const bool src_ok = !act || (a >= lo && r_mo + r_ml <= hi);
        if (span_ok && __all_sync(0xffffffffu, src_ok) && pidx && g_end - g_first <= kDoubleSpan) {
          // dense group: pointer jumping (see jump_span)
          span_jump(g_first, g_end - g_first, base, cnt);
          if (tm && t == 0) tm[7] += 1;
          continue;
        }
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
        if (ml <= 32 && mo + ml <= hi && fl + kRingChunk > mo && a + kRing >= hi && a >= vlo) {
          // fast path: no ring traffic, one pass, source inside the ring
          uint32_t r = t - off * __float2uint_rz(__fdividef((float)t + 0.5f, (float)off));
          r = off >= ml ? t : r;
          const uint8_t v = ring[(a + r) & (kRing - 1)];
          if (t < ml) ring[(mo + t) & (kRing - 1)] = v;
          __syncwarp();
          continue;
        }
        bool moved = skip_final(mo);
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
        const uint32_t lo = max(hi > kRing ? hi - kRing : 0u, vlo);
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
  __syncwarp();
  if (nthr > 32) {  // release the helper warps
    if (t == 0) cmd[0] = 0;
    bar_jump(nthr);  // B1
  }
  if (tm && t == 0) tm[4] = clock64();
}

// Whole page with the whole CTA (phases 1-4; phase 4 on warp 0).  Phase 4
// reuses the skim's tables (dead by then): the jump index at ctl + 72, the
// ring after it.
static_assert(72 + kDoubleSpan + kRing / 4 <= kSmemWords, "phase-4 ring must fit in ctl");
__device__ inline int32_t decode_block(const uint8_t* __restrict__ src, uint32_t n,
                                       uint8_t* __restrict__ dst, uint32_t raw_len, Scratch sc,
                                       uint32_t* ctl, long long* tm = nullptr) {
  const int32_t st = decode_prefix(src, n, dst, raw_len, sc, ctl, tm);
  if (st != kOk) return st;
  uint8_t* ring = reinterpret_cast<uint8_t*>(ctl + 72 + kDoubleSpan);
  if (threadIdx.x < 32) decode_matches(dst, raw_len, sc, ctl[1], ring, ctl + 72, tm);
  __syncthreads();
  return kOk;
}

}  // namespace lz4p
}  // namespace pcp
