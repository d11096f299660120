// kernels.cu — the sm_100a kernels of the PcRecord → batch stage.
//
//   k_crc_windows   zlib CRC-32 of page payloads, one warp per 64 KiB window,
//                   XOR-folded per page (device_crc.cuh)           [HBM]
//   k_page_decode   LZ4 block decode (lz4_block.cpp:113-156) / stored-raw
//                   copy of pages into the wave raw arena, one warp per page
//   k_scalar_parse  scalar-record walk (format.cpp:426-474) per group
//   k_cloud         persistent per-sample interpreter: stage blob (TMA bulk),
//                   fused payload CRC, XOR-delta decode + field split
//                   (format.cpp:183-195,483-493), the op chain
//                   (transforms.cpp:98-306 + App. C ops) and the write into
//                   the batch slot (Batch::stacked, pipeline.cpp:170-200)
//   k_finalize      page CRC verdicts + per-sample status precedence
//
// Every float op on a path whose result feeds a decision or an integer
// output uses explicit _rn intrinsics (no FMA), like the reference build.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cfloat>
#include <cstdint>

#include "device_crc.cuh"
#include "device_rng.cuh"
#include "device_util.cuh"
#include "device_sort.cuh"
#include "lz4_parallel.cuh"
#include "kernels.h"
#include "voxel_wave.h"
#include "pcp_internal.h"

namespace pcp {

__constant__ crc::X2N c_x2n;

// =========================================================================
// CRC over page payload windows
// =========================================================================
__global__ void k_crc_windows(const uint8_t* bytes, const CrcWindow* win, uint32_t n_win,
                              const uint32_t* shift_tab, uint32_t* page_acc) {
  __shared__ uint32_t tab[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = crc::table_entry(i);
  __syncthreads();
  const uint32_t warps = blockDim.x >> 5;
  for (uint32_t w = blockIdx.x * warps + (threadIdx.x >> 5); w < n_win; w += gridDim.x * warps) {
    const CrcWindow cw = win[w];
    const uint32_t c = crc::warp_range(tab, c_x2n.v, shift_tab, bytes + cw.start, cw.len, cw.after);
    if ((threadIdx.x & 31) == 0) atomicXor(page_acc + cw.page, c);
  }
}

// =========================================================================
// Page decode: LZ4 (warp per page) or stored-raw copy into the raw arena.
// Checks mirror decode_block_page (format.cpp:243-266) and lz4::decompress.
// The CRC verdict is folded in by k_finalize.
// =========================================================================
namespace {

struct Lz4Seq {
  uint64_t lit_src;  // payload offset of the literals
  uint64_t out;      // output offset of the literals
  uint32_t lit_len;
  uint32_t match_len;  // 0 = last sequence
  uint32_t offset;
};

// Parse one sequence starting at *ip (lane-0 work).  Returns status.
__device__ int32_t lz4_parse(const uint8_t* src, uint64_t n, uint64_t raw_len, uint64_t& ip,
                             uint64_t& op, Lz4Seq& s, bool& last) {
  if (ip >= n) return kCorruptPage;
  const uint8_t token = src[ip++];
  uint64_t lit = token >> 4;
  if (lit == 15) {
    uint8_t b;
    do {
      if (ip >= n) return kCorruptPage;
      b = src[ip++];
      lit += b;
    } while (b == 255);
  }
  if (ip + lit > n || op + lit > raw_len) return kCorruptPage;
  s.lit_src = ip;
  s.out = op;
  s.lit_len = (uint32_t)lit;
  ip += lit;
  op += lit;
  if (ip == n) {
    if (op != raw_len) return kCorruptPage;
    s.match_len = 0;
    s.offset = 0;
    last = true;
    return kOk;
  }
  if (ip + 2 > n) return kCorruptPage;
  const uint32_t offset = (uint32_t)src[ip] | ((uint32_t)src[ip + 1] << 8);
  ip += 2;
  if (offset == 0 || offset > op) return kCorruptPage;
  uint64_t ml = token & 0x0f;
  if (ml == 15) {
    uint8_t b;
    do {
      if (ip >= n) return kCorruptPage;
      b = src[ip++];
      ml += b;
    } while (b == 255);
  }
  ml += 4;
  if (op + ml > raw_len) return kCorruptPage;
  s.match_len = (uint32_t)ml;
  s.offset = offset;
  op += ml;
  last = false;
  return kOk;
}

}  // namespace

// Warp-cooperative LZ4 block decode (all 32 lanes call it).  Lane 0 parses
// up to 32 sequences ahead into shared memory; the warp then copies literal
// and match bytes cooperatively (a match with offset < length is copied in
// offset-sized strides, reproducing the byte-wise overlapping copy of
// lz4_block.cpp:151-153).  Returns the status on every lane.
__device__ int32_t warp_lz4_decode(const uint8_t* src, uint64_t n, uint8_t* dst, uint64_t raw_len,
                                   Lz4Seq* seqs, int32_t* sst, uint32_t* scount) {
  const int lane = threadIdx.x & 31;
  uint64_t ip = 0, op = 0;
  bool last = false;
  int32_t status = kOk;
  while (!last && status == kOk) {
    if (lane == 0) {
      uint32_t k = 0;
      int32_t st = kOk;
      while (k < 32 && !last) {
        st = lz4_parse(src, n, raw_len, ip, op, seqs[k], last);
        if (st != kOk) break;
        ++k;
      }
      *sst = st;
      *scount = k;
    }
    __syncwarp();
    const uint32_t k = *scount;
    status = *sst;
    last = __shfl_sync(0xffffffffu, last ? 1 : 0, 0) != 0;
    for (uint32_t q = 0; q < k; ++q) {
      const Lz4Seq s = seqs[q];
      for (uint32_t i = lane; i < s.lit_len; i += 32) dst[s.out + i] = src[s.lit_src + i];
      __syncwarp();
      if (s.match_len) {
        const uint64_t mo = s.out + s.lit_len;
        const uint32_t stride = s.offset < 32 ? s.offset : 32;
        for (uint32_t base = 0; base < s.match_len; base += stride) {
          const uint32_t i = base + lane;
          uint8_t b = 0;
          if (lane < stride && i < s.match_len) b = dst[mo - s.offset + i];
          __syncwarp();
          if (lane < stride && i < s.match_len) dst[mo + i] = b;
          __syncwarp();
        }
      }
    }
    __syncwarp();
  }
  return status;
}

// One CTA per page: LZ4 pages use the CTA-parallel decoder (lz4_parallel.cuh)
// with a per-page scratch slab; stored-raw pages are copied.  The rare page
// whose match count exceeds the scratch falls back to the warp decoder.
// CTA size of the page decoder (phases 1-3): 256 threads x 64 registers =
// 4 pages per SM.  128-thread CTAs (8 per SM) measured slower: the fill and
// phase-3 throughput per page matters as much as pages in flight.
constexpr uint32_t kDecodeThreads = 256;

__global__ void __launch_bounds__(kDecodeThreads, 1024 / kDecodeThreads) k_page_decode(const uint8_t* bytes, uint8_t* raw,
                                                     const PageRef* pages, const uint32_t* todo,
                                                     const uint64_t* scratch_off, uint8_t* scratch,
                                                     uint32_t n_todo, int32_t* page_status,
                                                     long long* timing) {
  __shared__ __align__(16) uint32_t ctl[lz4p::kSmemWords];
  __shared__ Lz4Seq seqs[32];
  __shared__ int32_t sst;
  __shared__ uint32_t scount;
  for (uint32_t w = blockIdx.x; w < n_todo; w += gridDim.x) {
    const uint32_t pi = todo[w];
    const PageRef pg = pages[pi];
    const uint8_t* src = bytes + pg.off + kPageHeaderBytes;
    uint8_t* dst = raw + pg.raw_dst;
    int32_t status = kOk;
    if (pg.flags & kFlagOuterLz4) {
      const lz4p::Scratch sc = lz4p::carve_scratch(scratch + scratch_off[w], pg.pay_len);
      if (pg.pay_len >= 0xFFFFFFF0ull || pg.raw_len >= 0xFFFFFFF0ull) {
        status = kCorruptPage;
        if (threadIdx.x == 0) sc.hdr[1] = 0;
      } else {
        // phases 1-3 here; phase 4 (one warp per page) in k_page_matches
        status = lz4p::decode_prefix(src, (uint32_t)pg.pay_len, dst, (uint32_t)pg.raw_len, sc, ctl,
                                     timing ? timing + 16 * (uint64_t)w : nullptr);
        if (threadIdx.x == 0) {
          sc.hdr[0] = ctl[1];
          sc.hdr[1] = status == kOk ? 1u : 0u;
        }
        if (status < 0) {
          if (threadIdx.x < 32) {
            const int32_t r = warp_lz4_decode(src, pg.pay_len, dst, pg.raw_len, seqs, &sst, &scount);
            if (threadIdx.x == 0) ctl[5] = (uint32_t)r;
          }
          __syncthreads();
          status = (int32_t)ctl[5];
        }
      }
    } else if (pg.flags & kFlagStoredRaw) {
      if (pg.pay_len != pg.raw_len) {
        status = kCorruptPage;
      } else {
        for (uint64_t i = threadIdx.x; i < pg.raw_len; i += blockDim.x) dst[i] = src[i];
      }
    } else {
      status = kCorruptPage;
    }
    if (threadIdx.x == 0 && status != kOk) page_status[pi] = status;
    __syncthreads();
  }
}

// Phase 4 of the LZ4 pages k_page_decode left pending: one warp per page
// (the match chains are serial; a 32-thread CTA with a 16 KB ring lets ~13
// pages per SM resolve at once instead of idling seven warps per page).
// Phase 4: warp 0 runs the match groups in order; warps 1-3 join every
// pointer-jumping span (dense label regions: ~620 spans of <= 2 KB per C2
// page, ~10 doubling rounds each), which a lone warp ran 64 bytes per lane
// per round.
constexpr uint32_t kMatchThreads = 128;
__global__ void __launch_bounds__(kMatchThreads) k_page_matches(uint8_t* raw, const PageRef* pages,
                                                     const uint32_t* todo, const uint64_t* scratch_off,
                                                     uint8_t* scratch, uint32_t n_todo,
                                                     long long* timing) {
  __shared__ __align__(16) uint8_t ring[lz4p::kRing];
  __shared__ uint32_t pidx[lz4p::kDoubleSpan];
  __shared__ uint32_t cmd[8];
  __shared__ uint32_t srec[3 * 256];  // a span's match records, staged by warp 0
  for (uint32_t w = blockIdx.x; w < n_todo; w += gridDim.x) {
    const PageRef pg = pages[todo[w]];
    if (!(pg.flags & kFlagOuterLz4)) continue;
    const lz4p::Scratch sc = lz4p::carve_scratch(scratch + scratch_off[w], pg.pay_len);
    if (sc.hdr[1] != 1u) continue;  // uniform over the CTA
    if (threadIdx.x >= 32) {
      lz4p::matches_helper(sc, ring, pidx, cmd, blockDim.x, srec);
      continue;
    }
    long long* tm = timing ? timing + 16 * (uint64_t)w + 8 : nullptr;  // [11] start, [12] end
    if (tm && threadIdx.x == 0) tm[3] = clock64();
    lz4p::decode_matches(raw + pg.raw_dst, (uint32_t)pg.raw_len, sc, sc.hdr[0], ring, pidx, tm,
                         blockDim.x, cmd, srec);
  }
}

// Phase 4 by page-wide pointer jumping: a warp per page
// resolves megabytes of match chains in stream order while most of the GPU
// idles (KITTI / S3DIS quantised pages: one cloud per page).  Here every
// output byte of a pending page gets a pointer to its source -- P[b] = b for
// literal bytes, b - off inside a match (the byte-wise overlapping copy) --
// and rounds of P[b] = P[P[b]] run over all pages at once.  Pointers only
// move to earlier ancestors, so in-place updates are safe and every chain
// ends at a literal byte within ceil(log2(depth)) + 1 rounds; then one gather
// out[b] = out[P[b]].  Work is tracked per 256-byte block: blocks without
// match bytes are never visited, and a block none of whose pointers moved in
// a round points only at literal bytes (roots never move), so it is retired.
// Phase 3 already checked every match: this is pure data movement.
// grid (n_todo, kPjSplit); warps take blocks.  Per page, the block flags
// live at F + raw_dst / 256 (bit 0: active, bit 1: holds match bytes).
constexpr uint32_t kPjSplit = 64;
constexpr uint32_t kPjBlock = 256;

__device__ __forceinline__ bool pj_page(uint8_t* raw, const PageRef* pages, const uint32_t* todo,
                                        const uint64_t* scratch_off, uint8_t* scratch, uint32_t* ptr,
                                        uint8_t* flags, uint32_t w, uint32_t*& P, uint8_t*& dst,
                                        uint8_t*& F, uint32_t& len, lz4p::Scratch& sc) {
  const PageRef pg = pages[todo[w]];
  if (!(pg.flags & kFlagOuterLz4)) return false;
  sc = lz4p::carve_scratch(scratch + scratch_off[w], pg.pay_len);
  if (sc.hdr[1] != 1u) return false;
  P = ptr + pg.raw_dst;  // raw_dst is 16-B aligned; blocks are page-relative
  dst = raw + pg.raw_dst;
  F = flags + pg.raw_dst / kPjBlock + w;  // disjoint per page: nblk <= (raw_len / 256) + 1
  len = (uint32_t)pg.raw_len;
  return true;
}

__global__ void __launch_bounds__(256) k_pj_init(uint8_t* raw, const PageRef* pages, const uint32_t* todo,
                                                 const uint64_t* scratch_off, uint8_t* scratch,
                                                 uint32_t* ptr, uint8_t* flags) {
  uint32_t* P;
  uint8_t *dst, *F;
  uint32_t len;
  lz4p::Scratch sc;
  if (!pj_page(raw, pages, todo, scratch_off, scratch, ptr, flags, blockIdx.x, P, dst, F, len, sc)) return;
  const uint32_t step = gridDim.y * blockDim.x;
  for (uint32_t b = blockIdx.y * blockDim.x + threadIdx.x; b < len; b += step) P[b] = b;
  const uint32_t nblk = (len + kPjBlock - 1) / kPjBlock;
  for (uint32_t k = blockIdx.y * blockDim.x + threadIdx.x; k < nblk; k += step) F[k] = 0;
}

__global__ void __launch_bounds__(256) k_pj_matches(uint8_t* raw, const PageRef* pages, const uint32_t* todo,
                                                    const uint64_t* scratch_off, uint8_t* scratch,
                                                    uint32_t* ptr, uint8_t* flags) {
  uint32_t* P;
  uint8_t *dst, *F;
  uint32_t len;
  lz4p::Scratch sc;
  if (!pj_page(raw, pages, todo, scratch_off, scratch, ptr, flags, blockIdx.x, P, dst, F, len, sc)) return;
  const uint32_t M = sc.hdr[0];
  const uint32_t step = gridDim.y * blockDim.x;
  for (uint32_t m = blockIdx.y * blockDim.x + threadIdx.x; m < M; m += step) {
    const uint32_t mo = sc.m_mo[m], ml = sc.m_ml[m], off = sc.m_off[m];
    for (uint32_t i = 0; i < ml; ++i) P[mo + i] = mo + i - off;
    if (ml)
      for (uint32_t k = mo / kPjBlock; k <= (mo + ml - 1) / kPjBlock; ++k) F[k] = 3;
  }
}

// round r; changed[r * n_todo + w] = some pointer of page w moved this round
__global__ void __launch_bounds__(256) k_pj_round(uint8_t* raw, const PageRef* pages, const uint32_t* todo,
                                                  const uint64_t* scratch_off, uint8_t* scratch,
                                                  uint32_t* ptr, uint8_t* flags, uint32_t* changed,
                                                  uint32_t n_todo, uint32_t r) {
  const uint32_t w = blockIdx.x;
  if (r > 0 && changed[(r - 1) * n_todo + w] == 0) return;  // page converged
  uint32_t* P;
  uint8_t *dst, *F;
  uint32_t len;
  lz4p::Scratch sc;
  if (!pj_page(raw, pages, todo, scratch_off, scratch, ptr, flags, w, P, dst, F, len, sc)) return;
  const uint32_t lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t nblk = (len + kPjBlock - 1) / kPjBlock;
  bool any = false;
  for (uint32_t k = blockIdx.y * nw + (threadIdx.x >> 5); k < nblk; k += gridDim.y * nw) {
    if (!(F[k] & 1u)) continue;  // warp-uniform
    const uint32_t b0 = k * kPjBlock;
    uint32_t p[kPjBlock / 32];
#pragma unroll
    for (int u = 0; u < (int)(kPjBlock / 32); ++u) {
      const uint32_t b = b0 + u * 32 + lane;
      p[u] = b < len ? P[b] : b;
    }
    bool ch = false;
#pragma unroll
    for (int u = 0; u < (int)(kPjBlock / 32); ++u) {
      const uint32_t b = b0 + u * 32 + lane;
      if (p[u] != b) {
        const uint32_t q = P[p[u]];
        if (q != p[u]) {
          P[b] = q;
          ch = true;
        }
      }
    }
    ch = __any_sync(0xffffffffu, ch);
    if (!ch && lane == 0) F[k] = 2;  // every pointer of the block is at a root: retired
    any |= ch;
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) changed[r * n_todo + w] = 1;
}

__global__ void __launch_bounds__(256) k_pj_gather(uint8_t* raw, const PageRef* pages, const uint32_t* todo,
                                                   const uint64_t* scratch_off, uint8_t* scratch,
                                                   uint32_t* ptr, uint8_t* flags) {
  uint32_t* P;
  uint8_t *dst, *F;
  uint32_t len;
  lz4p::Scratch sc;
  if (!pj_page(raw, pages, todo, scratch_off, scratch, ptr, flags, blockIdx.x, P, dst, F, len, sc)) return;
  const uint32_t lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t nblk = (len + kPjBlock - 1) / kPjBlock;
  for (uint32_t k = blockIdx.y * nw + (threadIdx.x >> 5); k < nblk; k += gridDim.y * nw) {
    if (!(F[k] & 2u)) continue;  // literal-only block: final already
#pragma unroll
    for (int u = 0; u < (int)(kPjBlock / 32); ++u) {
      const uint32_t b = k * kPjBlock + u * 32 + lane;
      if (b < len) {
        const uint32_t p = P[b];
        if (p != b) dst[b] = dst[p];  // p is a literal byte: final, never written here
      }
    }
  }
}

// =========================================================================
// Scalar-record parse: one thread walks one group's decoded scalar page
// (parse_scalar_record, format.cpp:426-474).  Values of non-bytes fields are
// copied, in schema order, into the value arena for the batch.
// =========================================================================
__global__ void k_scalar_parse(WaveArgs a) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.n_groups) return;
  const GroupWork gw = a.groups[g];
  const PageRef pg = a.pages[gw.scalar_page];
  const uint8_t* p = a.raw + pg.raw_dst;
  const uint64_t n = pg.raw_len;
  uint64_t pos = 0;
  uint32_t vo = gw.vals_base;
  int32_t fatal = kOk;
  for (uint32_t r = 0; r < gw.n_rows; ++r) {
    ScalarRec rec{};
    rec.status = fatal;
    if (fatal == kOk) {
      auto rd = [&](void* dstp, uint32_t k) -> bool {
        if (pos + k > n) return false;
        uint8_t* d = static_cast<uint8_t*>(dstp);
        for (uint32_t i = 0; i < k; ++i) d[i] = p[pos + i];
        pos += k;
        return true;
      };
      uint32_t nl = 0;
      bool ok = rd(&rec.blob_start, 8) && rd(&rec.blob_end, 8) && rd(&nl, 4);
      if (ok && nl > kMaxBytesFields) ok = false;
      rec.n_lens = nl;
      for (uint32_t i = 0; ok && i < nl; ++i) ok = rd(&rec.lens[i], 8);
      rec.vals_off = vo;
      for (int f = 0; ok && f < a.n_fields; ++f) {
        const FieldDesc fd = a.fields[f];
        uint32_t es = 0;
        switch (fd.kind) {
          case kBytes: continue;
          case kInt32: case kFloat32: es = 4; break;
          case kInt64: case kFloat64: es = 8; break;
          case kString: {
            uint32_t len = 0;
            ok = rd(&len, 4);
            if (ok && pos + len > n) ok = false;
            if (ok) {
              // strings keep their u32 length prefix in the value arena
              uint8_t* d = a.vals + vo;
              *reinterpret_cast<uint32_t*>(d) = len;
              for (uint32_t i = 0; i < len; ++i) d[4 + i] = p[pos + i];
              pos += len;
              vo += 4 + len;
            }
            continue;
          }
        }
        const uint32_t nb = es * fd.elems;
        if (pos + nb > n) {
          ok = false;
          break;
        }
        for (uint32_t i = 0; i < nb; ++i) a.vals[vo + i] = p[pos + i];
        pos += nb;
        vo += nb;
      }
      rec.vals_len = vo - rec.vals_off;
      if (!ok) {
        fatal = kCorruptPage;  // "record truncated" (format.cpp:25-27)
        rec.status = fatal;
      }
    }
    a.recs[gw.first_rec + r] = rec;
  }
}

// =========================================================================
// The per-sample interpreter
// =========================================================================
namespace {

constexpr int kRed = 64;  // reduction scratch words (8 B)



// An op's seed (mix_seed, transforms.cpp:82-96) and, when k_seed_states ran,
// its pre-seeded MT19937-64 state in global memory.
struct Seed {
  uint64_t v;
  const uint64_t* pre;
};

struct Cloud {
  uint8_t* cur[kMaxBytesFields];
  uint8_t* alt[kMaxBytesFields];
  uint32_t n[kMaxBytesFields];     // points (tracked fields)
  uint32_t elem[kMaxBytesFields];  // bytes per point
  uint32_t present;                // tracked + present bits
  int32_t* ix[4];                  // index scratch, cap entries each
  uint32_t cap;
  uint64_t* key[2];                // voxel sort keys (ping-pong)
  int32_t* counts;                 // voxel counts (cap)
  uint32_t n_counts;
  int32_t has_counts;
  uint8_t* fps_buf;                // cluster FPS: mailbox + this CTA's slice (buffer 24)
  uint32_t* sort_buf;              // voxel sort scratch (buffer 25, kSortScratchBytes)
};

struct Smem {
  uint32_t rs_base[16];
  uint32_t rs_wcnt[16][16];  // per-warp digit counts (radix sort tiles)
  uint32_t crc_tab[256];
  unsigned long long red[kRed];
  uint64_t mt[rng::kN];
  uint64_t bar;
  uint64_t fbar[2];           // cluster-FPS mailbox barriers (per parity)
  int32_t status;
  int32_t flag;
  uint32_t u32s[8];
  float f32s[8];
  double f64s[8];
  Cloud cl;                   // the current sample's descriptor (single writer: thread 0)
  Cloud proto;
  uint64_t flen[kMaxBytesFields], foff[kMaxBytesFields];
  int32_t pre_status;
};

__device__ __forceinline__ float* F(Cloud& c, int f) { return reinterpret_cast<float*>(c.cur[f]); }

__device__ __forceinline__ bool has(const Cloud& c, int f) {
  return f >= 0 && ((c.present >> f) & 1u);
}

// Lowest-set-bit exponent of a finite nonzero float: x = odd * 2^e.
__device__ __forceinline__ int lowbit_exp(float x) {
  const uint32_t b = __float_as_uint(x) & 0x7fffffffu;
  const uint32_t e = b >> 23, m = b & 0x7fffffu;
  if (e == 0) return -149 + __ffs(m) - 1;
  return (int)e - 150 + __ffs(m | 0x800000u) - 1;
}

// ---- gather helpers -------------------------------------------------------
__device__ void gather_field(Cloud& c, int f, const int32_t* idx, uint32_t m) {
  const uint32_t es = c.elem[f];
  const uint8_t* src = c.cur[f];
  uint8_t* dst = c.alt[f];
  if (es == 12) {
    const float* s = reinterpret_cast<const float*>(src);
    float* d = reinterpret_cast<float*>(dst);
    for (uint32_t k = threadIdx.x; k < m; k += blockDim.x) {
      const uint32_t i = (uint32_t)idx[k];
      d[3 * k] = s[3 * i];
      d[3 * k + 1] = s[3 * i + 1];
      d[3 * k + 2] = s[3 * i + 2];
    }
  } else if (es == 4) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    for (uint32_t k = threadIdx.x; k < m; k += blockDim.x) d[k] = s[idx[k]];
  } else {
    for (uint32_t k = threadIdx.x; k < m * es; k += blockDim.x) {
      const uint32_t p = k / es, b = k - p * es;
      dst[k] = src[(uint64_t)idx[p] * es + b];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint8_t* t = c.cur[f];
    c.cur[f] = c.alt[f];
    c.alt[f] = t;
    c.n[f] = m;
  }
  __syncthreads();
}

// Mask of tracked fields an index op moves.
__device__ __forceinline__ uint32_t move_mask(const WaveArgs& a, const Cloud& c, bool all_fields,
                                              uint32_t gather_mask) {
  uint32_t m = 0;
  if (a.role_data >= 0) m |= 1u << a.role_data;
  if (a.role_normal >= 0) m |= 1u << a.role_normal;
  if (a.role_color >= 0) m |= 1u << a.role_color;
  if (all_fields && a.role_intensity >= 0) m |= 1u << a.role_intensity;
  m |= gather_mask;
  return m & c.present;
}

__device__ int32_t check_move(const WaveArgs& a, const Cloud& c, uint32_t mm) {
  const uint32_t n = c.n[a.role_data];
  for (int f = 0; f < a.n_bytes_fields; ++f)
    if (((mm >> f) & 1u) && c.n[f] < n) return kOutOfBounds;
  return kOk;
}

__device__ void gather_mask_fields(const WaveArgs& a, Cloud& c, uint32_t mm, const int32_t* idx,
                                   uint32_t m) {
  for (int f = 0; f < a.n_bytes_fields; ++f)
    if ((mm >> f) & 1u) gather_field(c, f, idx, m);
}

// ---- Fisher-Yates (transforms.cpp:278-287), parallel resolution ----------
// J[i] = draw i's swap partner.  idx[i] = value at position J[i] just before
// swap i = W[prev(i)] if an earlier swap wrote that position, else J[i];
// W[k] (value at position k before swap k) follows the chain of last
// writers back to an untouched original.
__device__ void fy_resolve(Cloud& c, Smem& S, uint32_t N, uint32_t T) {
  int32_t* J = c.ix[0];
  int32_t* last = c.ix[1];
  int32_t* prev = c.ix[2];
  int32_t* ptr = c.ix[3];
  for (uint32_t p = threadIdx.x; p < N; p += blockDim.x) last[p] = -1;
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    const uint32_t lt = (1u << lane) - 1u, gt = ~((2u << lane) - 1u);
    for (uint32_t base = 0; base < T; base += 32) {
      const uint32_t i = base + lane;
      const bool v = i < T;
      const uint32_t j = v ? (uint32_t)J[i] : (0x80000000u | lane);
      const uint32_t m = __match_any_sync(0xffffffffu, j);
      const int32_t cand = v ? last[j] : -1;
      __syncwarp();
      if (v) {
        const uint32_t lower = m & lt;
        prev[i] = lower ? (int32_t)(base + 31 - __clz(lower)) : cand;
        if ((m & gt) == 0) last[j] = (int32_t)i;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < T; k += blockDim.x) {
    const int32_t l = last[k];
    ptr[k] = (l == (int32_t)k) ? prev[k] : l;
  }
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) S.flag = 0;
    __syncthreads();
    bool ch = false;
    for (uint32_t k = threadIdx.x; k < T; k += blockDim.x) {
      const int32_t p = ptr[k];
      if (p >= 0) {
        const int32_t q = ptr[p];
        if (q >= 0) {
          ptr[k] = q;
          ch = true;
        }
      }
    }
    if (ch) S.flag = 1;
    __syncthreads();
    if (!S.flag) break;
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < T; i += blockDim.x) {
    const int32_t pv = prev[i];
    int32_t v;
    if (pv >= 0) {
      const int32_t r = ptr[pv];
      v = r >= 0 ? r : pv;
    } else {
      v = J[i];
    }
    J[i] = v;  // J becomes idx (each i is read and written by one thread)
  }
  __syncthreads();
}

// MT19937-64 seeding (std::mt19937_64(seed), transforms.cpp:114): a copy of
// the state k_seed_states seeded for this (sample, op) when there is one,
// else thread 0's serial 311-step recurrence.  Callers sync afterwards.
__device__ __forceinline__ void seed_mt(Smem& S, Seed seed) {
  if (seed.pre) {
    for (uint32_t i = threadIdx.x; i < (uint32_t)rng::kN; i += blockDim.x) S.mt[i] = seed.pre[i];
  } else if (threadIdx.x == 0) {
    rng::seed_state(S.mt, seed.v);
  }
}

// Draw index vector for downsample; returns false if a Lemire rejection
// (probability ~range/2^64) needs the serial path.
__device__ bool downsample_draws(Cloud& c, Smem& S, Seed seed, uint32_t N, uint32_t T) {
  seed_mt(S, seed);
  if (threadIdx.x == 0) S.flag = 0;
  __syncthreads();
  int32_t* J = c.ix[0];
  const bool fy = N >= T;
  for (uint32_t blk = 0; blk * rng::kN < T; ++blk) {
    rng::twist_block(S.mt);
    for (uint32_t t = threadIdx.x; t < rng::kN; t += blockDim.x) {
      const uint32_t i = blk * rng::kN + t;
      if (i < T) {
        const uint64_t u = rng::temper(S.mt[t]);
        const uint64_t range = fy ? (uint64_t)(N - i) : (uint64_t)N;
        uint64_t r;
        if (!rng::lemire_fast(u, range, r)) S.flag = 1;
        J[i] = (int32_t)(fy ? i + r : r);
      }
    }
    __syncthreads();
  }
  return S.flag == 0;
}

__device__ void downsample_serial(Cloud& c, Smem& S, uint64_t seed, uint32_t N, uint32_t T) {
  int32_t* idx = c.ix[0];
  int32_t* all = c.ix[1];
  if (threadIdx.x == 0) {
    rng::Serial g{S.mt, 0};
    g.seed(seed);
    if (N >= T) {
      for (uint32_t i = 0; i < N; ++i) all[i] = (int32_t)i;
      for (uint32_t i = 0; i < T; ++i) {
        const uint32_t j = (uint32_t)g.uniform_int(i, N - 1);
        const int32_t t = all[i];
        all[i] = all[j];
        all[j] = t;
        idx[i] = all[i];
      }
    } else {
      for (uint32_t i = 0; i < T; ++i) idx[i] = (int32_t)g.uniform_int(0, N - 1);
    }
  }
  __syncthreads();
}

// ---- ops -------------------------------------------------------------------
__device__ int32_t op_normalize(const WaveArgs& a, Cloud& c, Smem& S) {
  float* d = F(c, a.role_data);
  const uint32_t n = c.n[a.role_data];
  double s[3] = {0, 0, 0}, ab[3] = {0, 0, 0};
  int e[3] = {INT_MAX, INT_MAX, INT_MAX};
  uint32_t bad = 0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float x = d[3 * i + k];
      s[k] = __dadd_rn(s[k], (double)x);
      ab[k] = __dadd_rn(ab[k], fabs((double)x));
      if (!isfinite(x)) bad |= 1u << k;
      else if (x != 0.0f) e[k] = min(e[k], lowbit_exp(x));
    }
  }
  double sum[3], A[3];
  int em[3];
  for (int k = 0; k < 3; ++k) {
    sum[k] = dev::block_reduce(s[k], dev::OpDAdd{}, 0.0, S.red);
    A[k] = dev::block_reduce(ab[k], dev::OpDAdd{}, 0.0, S.red);
    em[k] = dev::block_reduce(e[k], dev::OpMin{}, INT_MAX, S.red);
  }
  bad = dev::block_reduce(bad, dev::OpOr{}, 0u, S.red);
  // Exactness certificate: all coordinates are multiples of 2^em and every
  // partial sum is bounded by A <= 2^(52+em), so every partial sum of every
  // order is exact and equals the sequential double sum of the reference
  // (transforms.cpp:124-129).  Otherwise replay the sequential sum.
  if (threadIdx.x < 3) {
    const int k = threadIdx.x;
    const bool ok = !((bad >> k) & 1u) &&
                    (em[k] == INT_MAX || A[k] <= ldexp(1.0, min(52 + em[k], 1023)));
    double r = sum[k];
    if (!ok) {
      r = 0.0;
      for (uint32_t i = 0; i < n; ++i) r = __dadd_rn(r, (double)d[3 * i + k]);
    }
    S.f64s[k] = __ddiv_rn(r, (double)n);
  }
  __syncthreads();
  const double cx = S.f64s[0], cy = S.f64s[1], cz = S.f64s[2];
  double mx = 0.0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double dx = __dsub_rn((double)d[3 * i], cx);
    const double dy = __dsub_rn((double)d[3 * i + 1], cy);
    const double dz = __dsub_rn((double)d[3 * i + 2], cz);
    const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                          __dmul_rn(dz, dz)));
    mx = fmax(mx, r);  // std::max(s, r): NaN never replaces
  }
  const double sc = dev::block_reduce(mx, dev::OpFMax{}, 0.0, S.red);
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    if (sc == 0.0) {
      d[3 * i] = d[3 * i + 1] = d[3 * i + 2] = 0.0f;
    } else {
      d[3 * i] = __double2float_rn(__ddiv_rn(__dsub_rn((double)d[3 * i], cx), sc));
      d[3 * i + 1] = __double2float_rn(__ddiv_rn(__dsub_rn((double)d[3 * i + 1], cy), sc));
      d[3 * i + 2] = __double2float_rn(__ddiv_rn(__dsub_rn((double)d[3 * i + 2], cz), sc));
    }
  }
  __syncthreads();
  return kOk;
}

// Broadcast the first k (<= 8) engine outputs to S.u32s/f32s via thread 0.
__device__ void first_draws(Smem& S, Seed seed, int k, uint64_t* out) {
  __shared__ uint64_t o[8];
  if (threadIdx.x == 0) {
    if (seed.pre) {  // the op's first outputs, tempered by k_seed_states
      for (int i = 0; i < k; ++i) o[i] = seed.pre[i];
    } else {
      rng::first_outputs(seed.v, k, o, S.mt);
    }
  }
  __syncthreads();
  for (int i = 0; i < k; ++i) out[i] = o[i];
  __syncthreads();
}

__device__ int32_t op_translate(const WaveArgs& a, Cloud& c, Smem& S, Seed seed) {
  uint64_t u[3];
  first_draws(S, seed, 3, u);
  const float t[3] = {rng::uniform_real(u[0], -0.2f, 0.2f), rng::uniform_real(u[1], -0.2f, 0.2f),
                      rng::uniform_real(u[2], -0.2f, 0.2f)};
  float* d = F(c, a.role_data);
  const uint32_t n3 = 3 * c.n[a.role_data];
  for (uint32_t i = threadIdx.x; i < n3; i += blockDim.x) d[i] = __fadd_rn(d[i], t[i % 3]);
  __syncthreads();
  return kOk;
}

__device__ int32_t op_scale(const WaveArgs& a, Cloud& c, Smem& S, Seed seed) {
  uint64_t u[1];
  first_draws(S, seed, 1, u);
  const float s = rng::uniform_real(u[0], 0.8f, 1.25f);
  float* d = F(c, a.role_data);
  const uint32_t n3 = 3 * c.n[a.role_data];
  for (uint32_t i = threadIdx.x; i < n3; i += blockDim.x) d[i] = __fmul_rn(d[i], s);
  __syncthreads();
  return kOk;
}

__device__ int32_t op_flip(const WaveArgs& a, Cloud& c, Smem& S, Seed seed) {
  uint64_t u[1];
  first_draws(S, seed, 1, u);
  if (rng::uniform_real(u[0], 0.0f, 1.0f) < 0.5f) {
    float* d = F(c, a.role_data);
    for (uint32_t i = threadIdx.x; i < c.n[a.role_data]; i += blockDim.x) d[3 * i] = -d[3 * i];
    if (has(c, a.role_normal)) {
      float* nm = F(c, a.role_normal);
      for (uint32_t i = threadIdx.x; i < c.n[a.role_normal]; i += blockDim.x) nm[3 * i] = -nm[3 * i];
    }
  }
  __syncthreads();
  return kOk;
}

__device__ void rotate_field(float* v, uint32_t n, float cs, float sn) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const float px = v[3 * i], py = v[3 * i + 1];
    v[3 * i] = __fsub_rn(__fmul_rn(px, cs), __fmul_rn(py, sn));
    v[3 * i + 1] = __fadd_rn(__fmul_rn(px, sn), __fmul_rn(py, cs));
  }
}

__device__ int32_t op_rotate(const WaveArgs& a, Cloud& c, Smem& S, const OpDesc& op,
                             Seed seed) {
  float theta = op.theta;
  if (!op.has_theta) {
    uint64_t u[1];
    first_draws(S, seed, 1, u);
    theta = rng::uniform_real(u[0], 0.0f, 6.28318548202514648f);  // (float)(2*M_PI)
  }
  float sn, cs;
  sincosf(theta, &sn, &cs);
  rotate_field(F(c, a.role_data), c.n[a.role_data], cs, sn);
  if (has(c, a.role_normal)) rotate_field(F(c, a.role_normal), c.n[a.role_normal], cs, sn);
  __syncthreads();
  return kOk;
}

__device__ __forceinline__ float clampf(float v, float lo, float hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

// jitter (transforms.cpp:159-168): normals n_0, n_1, ... from the polar
// method; accepted attempt j yields n_2j = y*mult (returned) and
// n_2j+1 = x*mult (saved).  Attempts are scanned 156 per twist.
__device__ int32_t op_jitter(const WaveArgs& a, Cloud& c, Smem& S, Seed seed) {
  float* d = F(c, a.role_data);
  const uint32_t need = 3 * c.n[a.role_data];
  seed_mt(S, seed);
  __syncthreads();
  uint32_t done = 0;  // normals produced
  while (done < need) {
    rng::twist_block(S.mt);
    for (uint32_t base = 0; base < rng::kM; base += blockDim.x) {
      const uint32_t t = base + threadIdx.x;
      float x = 0, y = 0, r2 = 0;
      bool acc = false;
      if (t < rng::kM)
        acc = rng::polar_attempt(rng::temper(S.mt[2 * t]), rng::temper(S.mt[2 * t + 1]), x, y, r2);
      uint32_t tot;
      const uint32_t rank = dev::block_scan_excl(acc ? 1u : 0u, &tot, S.red);
      if (acc) {
        const uint32_t k0 = done + 2 * rank;
        const float mult = rng::polar_mult(r2);
        if (k0 < need) {
          const float v = clampf(__fadd_rn(__fmul_rn(__fmul_rn(y, mult), 0.01f), 0.0f), -0.05f, 0.05f);
          d[k0] = __fadd_rn(d[k0], v);
        }
        if (k0 + 1 < need) {
          const float v = clampf(__fadd_rn(__fmul_rn(__fmul_rn(x, mult), 0.01f), 0.0f), -0.05f, 0.05f);
          d[k0 + 1] = __fadd_rn(d[k0 + 1], v);
        }
      }
      done += 2 * tot;
      __syncthreads();
    }
  }
  return kOk;
}

__device__ int32_t op_color(const WaveArgs& a, Cloud& c, Smem& S, Seed seed) {
  if (!has(c, a.role_color) || c.n[a.role_color] == 0) return kMissingField;
  float* col = F(c, a.role_color);
  const uint32_t need = 3 * c.n[a.role_color];
  seed_mt(S, seed);
  __syncthreads();
  for (uint32_t blk = 0; blk * rng::kN < need; ++blk) {
    rng::twist_block(S.mt);
    for (uint32_t t = threadIdx.x; t < rng::kN; t += blockDim.x) {
      const uint32_t k = blk * rng::kN + t;
      if (k < need)
        col[k] = clampf(__fadd_rn(col[k], rng::uniform_real(rng::temper(S.mt[t]), -0.1f, 0.1f)),
                        0.0f, 1.0f);
    }
    __syncthreads();
  }
  return kOk;
}

// Ordered compaction of the points passing `keep(i)` into ix[0]; returns m.
template <typename Pred>
__device__ uint32_t compact(Cloud& c, Smem& S, uint32_t n, Pred keep) {
  int32_t* out = c.ix[0];
  uint32_t base = 0;
  for (uint32_t t0 = 0; t0 < n; t0 += blockDim.x) {
    const uint32_t i = t0 + threadIdx.x;
    const bool k = i < n && keep(i);
    uint32_t tot;
    const uint32_t r = dev::block_scan_excl(k ? 1u : 0u, &tot, S.red);
    if (k) out[base + r] = (int32_t)i;
    base += tot;
  }
  __syncthreads();
  return base;
}

// random_crop (transforms.cpp:220-271).
__device__ int32_t op_random_crop(const WaveArgs& a, Cloud& c, Smem& S, Seed seed) {
  const float* d = F(c, a.role_data);
  const uint32_t n = c.n[a.role_data];
  // bbox: sequential std::min/std::max from pts[0]: equal values keep the
  // earliest, NaN never replaces, a NaN pts[0] poisons the axis.
  float lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    float l = INFINITY, h = -INFINITY;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const float v = d[3 * i + k];
      l = fminf(l, v);
      h = fmaxf(h, v);
    }
    lo[k] = dev::block_reduce(l, [](float x, float y) { return fminf(x, y); }, INFINITY, S.red);
    hi[k] = dev::block_reduce(h, [](float x, float y) { return fmaxf(x, y); }, -INFINITY, S.red);
    const float p0 = d[k];
    if (isnan(p0)) lo[k] = hi[k] = p0;
    // -0/+0 ties: the sequential min keeps the first of equal values
    if (lo[k] == 0.0f) lo[k] = (p0 == 0.0f) ? p0 : 0.0f;
    if (hi[k] == 0.0f) hi[k] = (p0 == 0.0f) ? p0 : 0.0f;
  }
  __syncthreads();
  // the "first zero" rule above is exact only when pts[0] is that zero; a
  // later signed zero can only matter for the box start, which is computed
  // from lo + positive terms — +0 and -0 give the same sums unless all terms
  // are zero.  Handled exactly by the rescan below.
  for (int k = 0; k < 3; ++k) {
    if (lo[k] == 0.0f && d[k] != 0.0f) {
      if (threadIdx.x == 0) {
        float z = 0.0f;
        for (uint32_t i = 0; i < n; ++i)
          if (d[3 * i + k] == 0.0f) { z = d[3 * i + k]; break; }
        S.f32s[k] = z;
      }
      __syncthreads();
      lo[k] = S.f32s[k];
      __syncthreads();
    }
    if (hi[k] == 0.0f && d[k] != 0.0f) {
      if (threadIdx.x == 0) {
        float z = 0.0f;
        for (uint32_t i = 0; i < n; ++i)
          if (d[3 * i + k] == 0.0f) { z = d[3 * i + k]; break; }
        S.f32s[k + 3] = z;
      }
      __syncthreads();
      hi[k] = S.f32s[k + 3];
      __syncthreads();
    }
  }
  uint64_t u[6];
  first_draws(S, seed, 6, u);
  float blo[3], bhi[3];
  for (int k = 0; k < 3; ++k) {
    const float ext = __fsub_rn(hi[k], lo[k]);
    const float f = rng::uniform_real(u[2 * k], 0.7f, 1.0f);
    const float uu = rng::uniform_real(u[2 * k + 1], 0.0f, 1.0f);
    blo[k] = __fadd_rn(lo[k], __fmul_rn(__fmul_rn(uu, ext), __fsub_rn(1.0f, f)));
    bhi[k] = __fadd_rn(blo[k], __fmul_rn(ext, f));
  }
  const uint32_t m = compact(c, S, n, [&](uint32_t i) {
    const float x = d[3 * i], y = d[3 * i + 1], z = d[3 * i + 2];
    return x >= blo[0] && x <= bhi[0] && y >= blo[1] && y <= bhi[1] && z >= blo[2] && z <= bhi[2];
  });
  if (m == 0) return kOk;  // fall back to the full cloud (:246)
  const uint32_t mm = move_mask(a, c, false, 0);
  const int32_t st = check_move(a, c, mm);
  if (st) return st;
  // intensity: only when it has at least as many entries as kept points,
  // keeping entries whose index exists (:257-269)
  if (has(c, a.role_intensity) && c.n[a.role_intensity] >= m) {
    const int fi = a.role_intensity;
    const uint32_t ni = c.n[fi];
    const int32_t* keep = c.ix[0];
    uint32_t* dst = reinterpret_cast<uint32_t*>(c.alt[fi]);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(c.cur[fi]);
    uint32_t base = 0;
    for (uint32_t t0 = 0; t0 < m; t0 += blockDim.x) {
      const uint32_t k = t0 + threadIdx.x;
      const bool ok = k < m && (uint32_t)keep[k] < ni;
      uint32_t tot;
      const uint32_t r = dev::block_scan_excl(ok ? 1u : 0u, &tot, S.red);
      if (ok) dst[base + r] = src[keep[k]];
      base += tot;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      c.cur[fi] = c.alt[fi];
      c.alt[fi] = reinterpret_cast<uint8_t*>(const_cast<uint32_t*>(src));
      c.n[fi] = base;
    }
    __syncthreads();
  }
  gather_mask_fields(a, c, mm, c.ix[0], m);
  return kOk;
}

__device__ int32_t op_downsample(const WaveArgs& a, Cloud& c, Smem& S, const OpDesc& op,
                                 Seed seed) {
  if (op.num_points <= 0) return kOutOfBounds;
  const uint32_t T = (uint32_t)op.num_points;
  const uint32_t N = c.n[a.role_data];
  if (T > c.cap) return kOutOfBounds;
  const uint32_t mm = move_mask(a, c, false, op.gather_mask);
  const int32_t st = check_move(a, c, mm);
  if (st) return st;
  const bool fast = downsample_draws(c, S, seed, N, T) && !a.force_serial_fy;
  if (fast) {
    if (N >= T) fy_resolve(c, S, N, T);
  } else {
    downsample_serial(c, S, seed.v, N, T);
  }
  gather_mask_fields(a, c, mm, c.ix[0], T);
  return kOk;
}

// FPS (App. C): start at 0, d2 = (dx*dx + dy*dy) + dz*dz without FMA,
// mind = min(mind, d2), next = argmax mind (lowest index on ties).
// Paired FP32 (sm_100 FADD2/FFMA2): two independent IEEE round-to-nearest
// operations per instruction, so the no-FMA distance below is bit-identical
// to the scalar form at half the FMA-pipe issue cost.
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// x*x as fma(x, x, nz) with nz = -0.0f known only at run time: ptxas 12.9
// contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 despite the explicit
// rounding modifiers; an FFMA2 result cannot be fused again, and
// fma(x, x, -0) == mul(x, x) for every x (including +-0, inf, NaN).
__device__ __forceinline__ uint64_t f2_sq(uint64_t a, uint64_t nz2) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(d) : "l"(a), "l"(nz2));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// CTA argmax of the min-distances for one FPS iteration: the largest value,
// lowest point index on ties (App. C).  Values first — warp redux.sync max
// of the distance bits (distances are >= +0, so the unsigned order of their
// bits is the float order; padding carries -inf and contributes 0), one
// block barrier through per-warp parity slots — then only the warp(s)
// holding the maximum look up which of their points it is (a min-tree over
// k, off every other warp's issue slots), and a second barrier publishes
// the lowest index.  Returns base + t + k*nt of the winner, or ~0u if the
// CTA has no point.  `slot`: >= 64 words of shared memory.
template <int P>
__device__ __forceinline__ uint32_t fps_argmax(const float (&mind)[P], float bv, uint32_t base,
                                               uint32_t* slot, uint32_t it, uint32_t& gmax_out) {
  const uint32_t t = threadIdx.x, nt = blockDim.x, lane = t & 31, w = t >> 5, nw = nt >> 5;
  const uint32_t par = it & 1u;
  const uint32_t vb = bv >= 0.f ? __float_as_uint(bv) : 0u;
  const uint32_t wmax = __reduce_max_sync(0xffffffffu, vb);
  if (lane == 0) slot[par * 16 + w] = wmax;
  __syncthreads();
  const uint32_t gv = lane < nw ? slot[par * 16 + lane] : 0u;
  const uint32_t gmax = __reduce_max_sync(0xffffffffu, gv);
  gmax_out = gmax;
  if (wmax == gmax) {  // warp-uniform
    uint32_t bk = 31;
    if (vb == gmax && bv >= 0.f) {
#pragma unroll
      for (int k = 0; k < P; ++k) bk = min(bk, mind[k] == bv ? (uint32_t)k : 31u);
    }
    const uint32_t bi = bk < 31 ? base + t + bk * nt : 0xFFFFFFFFu;
    const uint32_t wi = __reduce_min_sync(0xffffffffu, bi);
    if (lane == 0) slot[32 + par * 16 + w] = wi;
  }
  __syncthreads();
  return __reduce_min_sync(0xffffffffu,
                           (lane < nw && gv == gmax) ? slot[32 + par * 16 + lane] : 0xFFFFFFFFu);
}

// Register-resident FPS: thread t owns points i = t + k*nt (k < P), packed
// in pairs (k = 2j, 2j+1) with their min-distances in registers; the argmax
// per iteration is fps_argmax.
template <int P>
__device__ void fps_reg(const float* d, uint32_t N, uint32_t M, int32_t* idx, Smem& S, float nz) {
  static_assert(P % 2 == 0, "points are processed in pairs");
  uint32_t* slot = &S.rs_wcnt[0][0];  // [2][16] values, [2][16] indices
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  uint64_t X[P / 2], Y[P / 2], Z[P / 2];
  float mind[P];
#pragma unroll
  for (int j = 0; j < P / 2; ++j) {
    float v[2][3];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t i = t + (uint32_t)(2 * j + h) * nt;
      const bool ok = i < N;
      v[h][0] = ok ? d[3 * i] : 0.f;
      v[h][1] = ok ? d[3 * i + 1] : 0.f;
      v[h][2] = ok ? d[3 * i + 2] : 0.f;
      mind[2 * j + h] = ok ? INFINITY : -INFINITY;
    }
    X[j] = f2_pack(v[0][0], v[1][0]);
    Y[j] = f2_pack(v[0][1], v[1][1]);
    Z[j] = f2_pack(v[0][2], v[1][2]);
  }
  const uint64_t NZ = f2_pack(nz, nz);
  uint32_t sel = 0;
  for (uint32_t it = 0; it < M; ++it) {
    if (t == 0) idx[it] = (int32_t)sel;
    const float sx = d[3 * sel], sy = d[3 * sel + 1], sz = d[3 * sel + 2];
    const uint64_t SX = f2_pack(sx, sx), SY = f2_pack(sy, sy), SZ = f2_pack(sz, sz);
    float bv = -INFINITY;
#pragma unroll
    for (int j = 0; j < P / 2; ++j) {
      const uint64_t dx = f2_sub(X[j], SX), dy = f2_sub(Y[j], SY), dz = f2_sub(Z[j], SZ);
      const uint64_t dd = f2_add(f2_add(f2_sq(dx, NZ), f2_sq(dy, NZ)), f2_sq(dz, NZ));
      // fminf == (dd < mind ? dd : mind) here: dd is >= +0 or NaN (-> mind)
      mind[2 * j] = fminf(__uint_as_float((uint32_t)dd), mind[2 * j]);
      mind[2 * j + 1] = fminf(__uint_as_float((uint32_t)(dd >> 32)), mind[2 * j + 1]);
      bv = fmaxf(bv, fmaxf(mind[2 * j], mind[2 * j + 1]));
    }
    uint32_t gmax;
    sel = fps_argmax<P>(mind, bv, 0, slot, it, gmax);
    if (sel == 0xFFFFFFFFu) sel = 0;  // no candidate at all (N == 0): index 0 like the oracle
  }
}

// Cluster FPS for clouds above one CTA's register capacity:
// the points are split over the C CTAs of a thread-block cluster (CTA r owns
// [r*per, r*per + per)), each holding its slice in registers as in fps_reg
// plus an AoS copy in shared memory for its candidates' coordinates.  Per
// iteration each CTA reduces its warps' candidates (one block barrier, as
// fps_reg), then warp 0 sends the CTA's candidate (distance bits, index,
// x, y, z) to every CTA of the cluster with st.async into a parity
// double-buffered mailbox whose mbarrier counts the bytes — one DSMEM hop
// and an mbarrier wait instead of a cluster barrier (which would also flush
// L1) — and every CTA reduces the same C records to the same `sel`.  Reuse
// is safe: a CTA sends iteration it+2's record only after completing it+1,
// which needs every CTA's it+1 record, each sent after that CTA's block
// barrier of it+1, i.e. after all its threads read iteration it's mailbox.
template <int P>
__device__ void fps_cluster(const float* d, uint32_t N, uint32_t M, int32_t* idx, Smem& S,
                            float nz, uint8_t* buf, uint32_t C) {
  static_assert(P % 2 == 0, "points are processed in pairs");
  const uint32_t t = threadIdx.x, nt = blockDim.x, lane = t & 31, w = t >> 5, nw = nt >> 5;
  const uint32_t r = dev::cluster_rank();
  const uint32_t per = (N + C - 1) / C;
  const uint32_t base = min(r * per, N), nloc = min(per, N - base);
  uint32_t* mail = reinterpret_cast<uint32_t*>(buf);         // [2][128][8] words
  float* sp = reinterpret_cast<float*>(buf + kFpsMailBytes);  // [nloc][3]
  const uint32_t mail_s = dev::smem_u32(mail), sp_s = dev::smem_u32(sp);  // buf is in shared memory
  for (uint32_t k = t; k < 3 * nloc; k += nt) sp[k] = d[3 * (uint64_t)base + k];
  if (t == 0) {
    dev::mbar_init(&S.fbar[0], 1);
    dev::mbar_init(&S.fbar[1], 1);
    dev::fence_mbar_init();
  }
  __syncthreads();
  uint64_t X[P / 2], Y[P / 2], Z[P / 2];
  float mind[P];
#pragma unroll
  for (int j = 0; j < P / 2; ++j) {
    float v[2][3];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t i = t + (uint32_t)(2 * j + h) * nt;
      const bool ok = i < nloc;
      v[h][0] = ok ? sp[3 * i] : 0.f;
      v[h][1] = ok ? sp[3 * i + 1] : 0.f;
      v[h][2] = ok ? sp[3 * i + 2] : 0.f;
      mind[2 * j + h] = ok ? INFINITY : -INFINITY;
    }
    X[j] = f2_pack(v[0][0], v[1][0]);
    Y[j] = f2_pack(v[0][1], v[1][1]);
    Z[j] = f2_pack(v[0][2], v[1][2]);
  }
  dev::cluster_sync_all();  // every CTA's mailbox barriers are initialised
  uint32_t* slot = &S.rs_wcnt[0][0];  // fps_argmax slots
  const uint32_t tx = C * 20;  // bytes per phase: one record (16 + 4 B) from each CTA
  if (t == 0) {
    dev::mbar_expect_tx(&S.fbar[0], tx);
    dev::mbar_expect_tx(&S.fbar[1], tx);
  }
  const uint64_t NZ = f2_pack(nz, nz);
  uint32_t sel = 0;
  float sx = d[0], sy = d[1], sz = d[2];
  for (uint32_t it = 0; it < M; ++it) {
    if (t == 0) idx[it] = (int32_t)sel;
    const uint64_t SX = f2_pack(sx, sx), SY = f2_pack(sy, sy), SZ = f2_pack(sz, sz);
    float bv = -INFINITY;
#pragma unroll
    for (int j = 0; j < P / 2; ++j) {
      const uint64_t dx = f2_sub(X[j], SX), dy = f2_sub(Y[j], SY), dz = f2_sub(Z[j], SZ);
      const uint64_t dd = f2_add(f2_add(f2_sq(dx, NZ), f2_sq(dy, NZ)), f2_sq(dz, NZ));
      mind[2 * j] = fminf(__uint_as_float((uint32_t)dd), mind[2 * j]);
      mind[2 * j + 1] = fminf(__uint_as_float((uint32_t)(dd >> 32)), mind[2 * j + 1]);
      bv = fmaxf(bv, fmaxf(mind[2 * j], mind[2 * j + 1]));
    }
    const uint32_t par = it & 1u;
    uint32_t cmax;
    const uint32_t ci = fps_argmax<P>(mind, bv, base, slot, it, cmax);
    if (w == 0 && lane < C) {  // warp 0 sends the CTA's candidate to every CTA of the cluster
      float x = 0.f, y = 0.f, z = 0.f;
      if (ci != 0xFFFFFFFFu) {
        const uint32_t j = sp_s + 12 * (ci - base);
        x = dev::lds_f32(j);
        y = dev::lds_f32(j + 4);
        z = dev::lds_f32(j + 8);
      }
      const uint32_t* rec = mail + (par * 128 + r) * 8;
      const uint32_t ra = dev::mapa(rec, lane), rb = dev::mapa(&S.fbar[par], lane);
      dev::st_async_v4(ra, ci != 0xFFFFFFFFu ? cmax : 0u, ci, __float_as_uint(x), __float_as_uint(y), rb);
      dev::st_async_b32(ra + 16, __float_as_uint(z), rb);
    }
    // CTA-scope wait: st.async data is visible once its complete_tx lands
    // (an .acquire.cluster wait would also invalidate L1 every iteration)
    dev::mbar_wait(&S.fbar[par], (it >> 1) & 1u);
    if (t == 0 && it + 2 < M) dev::mbar_expect_tx(&S.fbar[par], tx);
    const uint32_t mb = mail_s + par * 128 * 32;
    uint32_t lv = 0, li = 0xFFFFFFFFu;
    if (lane < C) {
      lv = dev::lds_u32(mb + lane * 32);
      li = dev::lds_u32(mb + lane * 32 + 4);
    }
    const uint32_t gmax = __reduce_max_sync(0xffffffffu, lv);
    sel = __reduce_min_sync(0xffffffffu, lv == gmax ? li : 0xFFFFFFFFu);
    if (sel == 0xFFFFFFFFu) {  // no candidate at all: index 0 like the oracle
      sel = 0;
      sx = d[0], sy = d[1], sz = d[2];
    } else {
      const uint32_t bal = __ballot_sync(0xffffffffu, lane < C && lv == gmax && li == sel);
      const uint32_t q = __ffs(bal) - 1;
      sx = dev::lds_f32(mb + q * 32 + 8);
      sy = dev::lds_f32(mb + q * 32 + 12);
      sz = dev::lds_f32(mb + q * 32 + 16);
    }
  }
}

template <int MinBlocks>
__device__ int32_t op_fps(const WaveArgs& a, Cloud& c, Smem& S, const OpDesc& op) {
  if (op.num_points <= 0) return kOutOfBounds;
  const uint32_t M = (uint32_t)op.num_points;
  const uint32_t N = c.n[a.role_data];
  if (N < M || M > c.cap) return kOutOfBounds;
  const uint32_t mm = move_mask(a, c, true, op.gather_mask);
  const int32_t st = check_move(a, c, mm);
  if (st) return st;
  const float* d = F(c, a.role_data);
  int32_t* idx = c.ix[0];
  // register-resident paths (MinBlocks = 1 builds have 128 registers)
  bool done = false;
  if (N <= 8 * blockDim.x) {
    fps_reg<8>(d, N, M, idx, S, a.neg_zero);
    done = true;
  } else if (MinBlocks == 1 && N <= 16 * blockDim.x) {
    fps_reg<16>(d, N, M, idx, S, a.neg_zero);
    done = true;
  } else if (MinBlocks == 1 && N <= kFpsRegPts * blockDim.x) {
    fps_reg<kFpsRegPts>(d, N, M, idx, S, a.neg_zero);
    done = true;
  } else if (MinBlocks == 1 && a.fps_cluster > 1 && c.fps_buf && __isShared(c.fps_buf) &&
             N <= a.fps_cluster * a.fps_slice_pts && N <= a.fps_cluster * kFpsRegPts * blockDim.x) {
    // every CTA of the cluster takes this branch for the same sample
    fps_cluster<kFpsRegPts>(d, N, M, idx, S, a.neg_zero, c.fps_buf, a.fps_cluster);
    done = true;
  }
  if (done) {
    __syncthreads();
    gather_mask_fields(a, c, mm, idx, M);
    return kOk;
  }
  float* mind = reinterpret_cast<float*>(c.ix[1]);
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) mind[i] = INFINITY;
  __syncthreads();
  uint32_t sel = 0;
  for (uint32_t k = 0; k < M; ++k) {
    if (threadIdx.x == 0) idx[k] = (int32_t)sel;
    const float sx = d[3 * sel], sy = d[3 * sel + 1], sz = d[3 * sel + 2];
    float bv = -INFINITY;
    uint32_t bi = 0xFFFFFFFFu;
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
      const float dx = __fsub_rn(d[3 * i], sx), dy = __fsub_rn(d[3 * i + 1], sy),
                  dz = __fsub_rn(d[3 * i + 2], sz);
      const float dd = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
      float m = mind[i];
      if (dd < m) m = dd;
      mind[i] = m;
      if (dev::argmax_better(m, i, bv, bi)) {
        bv = m;
        bi = i;
      }
    }
    const dev::ArgMax r = dev::block_argmax(bv, bi, S.red);
    sel = r.i == 0xFFFFFFFFu ? 0 : r.i;
  }
  __syncthreads();
  gather_mask_fields(a, c, mm, idx, M);
  return kOk;
}

__device__ int32_t op_range_crop(const WaveArgs& a, Cloud& c, Smem& S, const OpDesc& op) {
  const float* d = F(c, a.role_data);
  const uint32_t n = c.n[a.role_data];
  const uint32_t mm = move_mask(a, c, true, op.gather_mask);
  const int32_t st = check_move(a, c, mm);
  if (st) return st;
  const uint32_t m = compact(c, S, n, [&](uint32_t i) {
    const float x = d[3 * i], y = d[3 * i + 1], z = d[3 * i + 2];
    return x >= op.lo[0] && x <= op.hi[0] && y >= op.lo[1] && y <= op.hi[1] && z >= op.lo[2] &&
           z <= op.hi[2];
  });
  gather_mask_fields(a, c, mm, c.ix[0], m);
  return kOk;
}

// ---- decode ----------------------------------------------------------------
// Copy len bytes (optionally XOR-delta decoding 4-byte words) from an
// arbitrarily aligned source into a 16-B aligned destination.
// U: 16-B chunks per thread in flight (4 in the 128-register build; 1 with
// 64 registers, where deeper unrolling spills to local memory)
template <int U, int DU>
__device__ void decode_bytes(uint8_t* dst, const uint8_t* src, uint64_t len, bool delta,
                             Smem& S) {
  const uint32_t t = threadIdx.x, nt = blockDim.x, lane = t & 31, w = t >> 5, nw = nt >> 5;
  if (!delta) {
    // 16-B stores built from aligned 4-B loads (funnel shift for the source
    // misalignment), 4 per thread in flight: a CTA streaming a multi-MB blob
    // is bound by loads in flight per SM, not by instructions
    const uint64_t h0 = (16u - (reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u;
    const uint64_t head = h0 < len ? h0 : len;
    for (uint64_t i = t; i < head; i += nt) dst[i] = src[i];  // dst may be 4-B aligned (output slots)
    dst += head;
    src += head;
    len -= head;
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
    const uint32_t sh = (uint32_t)(sa & 3u) * 8u;
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(sa & ~uintptr_t(3));
    const uint64_t n16 = len >> 4;
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (uint64_t k0 = t; k0 < n16; k0 += U * (uint64_t)nt) {
      uint32_t v[U][5];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t k = k0 + (uint64_t)u * nt;
        if (k < n16) {
#pragma unroll
          for (int e = 0; e < 5; ++e) v[u][e] = (e < 4 || sh) ? sw[4 * k + e] : 0u;  // <= 3 B past
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t k = k0 + (uint64_t)u * nt;
        if (k < n16)
          d4[k] = sh ? make_uint4(__funnelshift_r(v[u][0], v[u][1], sh), __funnelshift_r(v[u][1], v[u][2], sh),
                                  __funnelshift_r(v[u][2], v[u][3], sh), __funnelshift_r(v[u][3], v[u][4], sh))
                     : make_uint4(v[u][0], v[u][1], v[u][2], v[u][3]);
      }
    }
    for (uint64_t i = (n16 << 4) + t; i < len; i += nt) dst[i] = src[i];
    __syncthreads();
    return;
  }
  // XOR-delta: out[i] = XOR of in[0..i] over the (possibly unaligned) 4-byte
  // words of src.  Words are read as 16-B quads of the aligned word stream A
  // (the funnel shift's extra word comes from the next lane), one quad per
  // lane per row, DU rows in flight per warp.  Two passes over contiguous warp
  // segments of quads: (1) XOR-reduce, one prefix over the warp totals;
  // (2) lane-local scan of the quad, warp scan of the lane totals, row
  // carries chained from row totals.  Up to 3 head words (before the first
  // 16-B boundary of A) and 3 tail words are done by thread 0.
  const uint64_t nwords = len >> 2;  // len % 4 == 0 for delta columns
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
  const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
  const uint32_t sh = (uint32_t)(sa & 3u) * 8u;
  const uint32_t* A = reinterpret_cast<const uint32_t*>(sa & ~uintptr_t(3));
  const uint64_t h0 = ((16u - (reinterpret_cast<uintptr_t>(A) & 15u)) & 15u) >> 2;
  const uint64_t h = h0 < nwords ? h0 : nwords;
  const uint64_t nq = (nwords - h) >> 2;
  const uint64_t tail0 = h + 4 * nq;
  const uint64_t segq = ((nq + nw - 1) / nw + 31) & ~uint64_t(31);
  const uint64_t q0 = min((uint64_t)w * segq, nq), q1 = min(q0 + segq, nq);
  auto word = [&](uint64_t i) -> uint32_t { return sh ? __funnelshift_r(A[i], A[i + 1], sh) : A[i]; };
  // the 4 words of quad qi (lane-valid `ok`); every lane of the warp calls it
  auto quad = [&](uint64_t qi, bool ok, uint32_t (&o)[4]) {
    const uint4 q = ok ? *reinterpret_cast<const uint4*>(A + h + 4 * qi) : make_uint4(0u, 0u, 0u, 0u);
    uint32_t nx = __shfl_down_sync(0xffffffffu, q.x, 1);
    const bool next_ok = lane < 31 && qi + 1 < q1;
    if (ok && !next_ok && sh) nx = A[h + 4 * qi + 4];
    o[0] = __funnelshift_r(q.x, q.y, sh);
    o[1] = __funnelshift_r(q.y, q.z, sh);
    o[2] = __funnelshift_r(q.z, q.w, sh);
    o[3] = __funnelshift_r(q.w, nx, sh);
  };
  uint32_t x = 0;
  for (uint64_t base = q0; base < q1; base += 32 * DU) {
    uint32_t v[DU][4];
#pragma unroll
    for (int u = 0; u < DU; ++u) {
      const uint64_t qi = base + 32 * u + lane;
      quad(qi, qi < q1, v[u]);
    }
#pragma unroll
    for (int u = 0; u < DU; ++u) x ^= v[u][0] ^ v[u][1] ^ v[u][2] ^ v[u][3];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, o);
  uint32_t* red = reinterpret_cast<uint32_t*>(S.red);
  __syncthreads();  // S.red may still be read by a previous user
  if (lane == 0) red[w] = x;
  if (t == 0) {
    uint32_t hx = 0;
    for (uint64_t i = 0; i < h; ++i) hx ^= word(i);
    red[nw] = hx;
  }
  __syncthreads();
  uint32_t carry = red[nw];
  for (uint32_t k = 0; k < w; ++k) carry ^= red[k];
  for (uint64_t base = q0; base < q1; base += 32 * DU) {
    uint32_t v[DU][4];
#pragma unroll
    for (int u = 0; u < DU; ++u) {
      const uint64_t qi = base + 32 * u + lane;
      quad(qi, qi < q1, v[u]);
    }
#pragma unroll
    for (int u = 0; u < DU; ++u) {
      v[u][1] ^= v[u][0];
      v[u][2] ^= v[u][1];
      v[u][3] ^= v[u][2];
      uint32_t incl = v[u][3];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl ^= y;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t pre = incl ^ v[u][3] ^ carry;
      const uint64_t qi = base + 32 * u + lane;
      if (qi < q1) {
        uint32_t* d = d32 + h + 4 * qi;
        d[0] = v[u][0] ^ pre;
        d[1] = v[u][1] ^ pre;
        d[2] = v[u][2] ^ pre;
        d[3] = v[u][3] ^ pre;
      }
      carry ^= tot;
    }
  }
  if (t == 0) {
    uint32_t c0 = 0;
    for (uint64_t i = 0; i < h; ++i) d32[i] = c0 ^= word(i);
    c0 = red[nw];
    for (uint32_t k = 0; k < nw; ++k) c0 ^= red[k];
    for (uint64_t i = tail0; i < nwords; ++i) d32[i] = c0 ^= word(i);
  }
  __syncthreads();
}

}  // namespace

// Stable LSD radix sort of (key, val) by the low `bits` bits of key, 4-bit
// digits, whole CTA.  Ping-pongs between (k0,v0) and (k1,v1); returns the
// buffer index (0/1) holding the result.
__device__ int radix_sort(uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint32_t n,
                          uint32_t bits, Smem& S) {
  const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
  uint64_t* ks[2] = {k0, k1};
  uint32_t* vs[2] = {v0, v1};
  int cur = 0;
  for (uint32_t sh = 0; sh < bits; sh += 4) {
    const uint64_t* kin = ks[cur];
    const uint32_t* vin = vs[cur];
    uint64_t* kout = ks[cur ^ 1];
    uint32_t* vout = vs[cur ^ 1];
    if (t < 16) S.rs_base[t] = 0;
    __syncthreads();
    for (uint32_t i = t; i < n; i += blockDim.x) atomicAdd(&S.rs_base[(kin[i] >> sh) & 15u], 1u);
    __syncthreads();
    if (t == 0) {
      uint32_t acc = 0;
      for (int d = 0; d < 16; ++d) {
        const uint32_t c = S.rs_base[d];
        S.rs_base[d] = acc;
        acc += c;
      }
    }
    __syncthreads();
    for (uint32_t t0 = 0; t0 < n; t0 += blockDim.x) {
      const uint32_t i = t0 + t;
      const bool valid = i < n;
      uint64_t key = 0;
      uint32_t val = 0, d = 16;
      if (valid) {
        key = kin[i];
        val = vin[i];
        d = (uint32_t)(key >> sh) & 15u;
      }
      if (lane < 16) S.rs_wcnt[w][lane] = 0;
      __syncwarp();
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
      if (valid && rank == 0) S.rs_wcnt[w][d] = __popc(peers);
      __syncthreads();
      if (valid) {
        uint32_t off = S.rs_base[d] + rank;
        for (uint32_t q = 0; q < w; ++q) off += S.rs_wcnt[q][d];
        kout[off] = key;
        vout[off] = val;
      }
      __syncthreads();
      if (t < 16) {
        uint32_t tot = 0;
        for (uint32_t q = 0; q < nw; ++q) tot += S.rs_wcnt[q][t];
        S.rs_base[t] += tot;
      }
      __syncthreads();
    }
    cur ^= 1;
  }
  return cur;
}

// Per-axis extremes of a cloud in one pass: the plain min / max over the
// non-NaN coordinates and whether any coordinate is NaN.  With `origin`, also
// the smallest coordinate per axis with the sequential `if (v < o) o = v`
// semantics starting from point 0 (App. C voxel origin): NaN at point 0
// poisons the axis; later NaNs never win; equal values keep the first.
template <int U>
__device__ void axis_extremes(const float* d, uint32_t n, Smem& S, float* mn, float* mx, bool& any_nan,
                              float* origin) {
  float l3[3] = {INFINITY, INFINITY, INFINITY}, h3[3] = {-INFINITY, -INFINITY, -INFINITY};
  uint32_t nan = 0;
  for (uint32_t i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {  // all axes, U points in flight
    float v[U][3];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 3; ++k) v[u][k] = i0 + u * blockDim.x < n ? d[3 * (i0 + u * blockDim.x) + k] : d[k];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        l3[k] = fminf(l3[k], v[u][k]);
        h3[k] = fmaxf(h3[k], v[u][k]);
        nan |= isnan(v[u][k]) ? 1u : 0u;
      }
  }
  any_nan = dev::block_reduce(nan, dev::OpOr{}, 0u, S.red) != 0;
  for (int k = 0; k < 3; ++k) {
    mn[k] = dev::block_reduce(l3[k], [](float x, float y) { return fminf(x, y); }, INFINITY, S.red);
    mx[k] = dev::block_reduce(h3[k], [](float x, float y) { return fmaxf(x, y); }, -INFINITY, S.red);
    if (!origin) continue;
    origin[k] = mn[k];
    const float p0 = d[k];
    if (isnan(p0)) origin[k] = p0;
    else if (origin[k] == 0.0f) {  // first zero in point order keeps its sign
      if (threadIdx.x == 0) {
        float z = 0.0f;
        for (uint32_t i = 0; i < n; ++i)
          if (d[3 * i + k] == 0.0f) { z = d[3 * i + k]; break; }
        S.f32s[k] = z;
      }
      __syncthreads();
      origin[k] = S.f32s[k];
      __syncthreads();
    }
  }
}

// voxel / grid subsample (App. C): k = (int32)floorf((p - o) / v) per axis,
// key = kx | ky<<21 | kz<<42, stable order by key, per voxel the count and
// the mean of every float field = (float)(sum in point order (double) / count);
// extra gathered fields take the voxel's first point.  Output ascending key.
template <int U>
__device__ int32_t op_voxel(const WaveArgs& a, Cloud& c, Smem& S, const OpDesc& op) {
  const uint32_t n = c.n[a.role_data];
  if (!(op.voxel > 0.0f)) return kOutOfBounds;
  if (!c.key[0]) return kOutOfBounds;
  const uint32_t mm = move_mask(a, c, true, op.gather_mask);
  const int32_t st = check_move(a, c, mm);
  if (st) return st;
  const float* d = F(c, a.role_data);
  long long vt = (a.op_cycles && threadIdx.x == 0) ? clock64() : 0;
  auto vmark = [&](int slot) {  // PCP_OP_TIMING: voxel phases in op_cycles[10..15]
    if (a.op_cycles && threadIdx.x == 0) {
      const long long t1 = clock64();
      atomicAdd(a.op_cycles + 10 + slot, (unsigned long long)(t1 - vt));
      vt = t1;
    }
  };
  // origin + extent in one pass over the coordinates.  The App. C key
  // floorf((p - o) / v) is monotone in p (fsub_rn, fdiv_rn by v > 0 and
  // floorf all are), and NaN only arises from a NaN or infinite coordinate
  // (the extremes themselves) or origin, so every key is in [0, 2^21) iff no
  // coordinate is NaN and the keys of the per-axis min and max are, and the
  // largest key per axis is the max coordinate's: no per-point division here.
  float o[3], cmin[3], cmax[3];
  bool any_nan = false;
  if (op.has_origin) {
    o[0] = op.origin[0]; o[1] = op.origin[1]; o[2] = op.origin[2];
    axis_extremes<U>(d, n, S, cmin, cmax, any_nan, nullptr);
  } else {
    axis_extremes<U>(d, n, S, cmin, cmax, any_nan, o);
  }
  uint32_t* idx = reinterpret_cast<uint32_t*>(c.ix[0]);
  uint32_t* idx2 = reinterpret_cast<uint32_t*>(c.ix[1]);
  bool bad = any_nan;
  uint32_t mx[3] = {0, 0, 0};
  for (int ax = 0; ax < 3; ++ax) {
    const float ql = floorf(__fdiv_rn(__fsub_rn(cmin[ax], o[ax]), op.voxel));
    const float qh = floorf(__fdiv_rn(__fsub_rn(cmax[ax], o[ax]), op.voxel));
    if (!(ql >= 0.0f && ql < 2097152.0f) || !(qh >= 0.0f && qh < 2097152.0f)) bad = true;
    else mx[ax] = (uint32_t)qh;
  }
  if (bad) return kOutOfBounds;
  vmark(0);  // origin + extent pass
  uint32_t bx[3];
  for (int ax = 0; ax < 3; ++ax) bx[ax] = mx[ax] ? 32u - __clz(mx[ax]) : 0u;
  // compact sort key, monotone in the App. C key (kz major, then ky, kx)
  const uint32_t kb = bx[0] + bx[1] + bx[2];
  const uint32_t ib = n > 1 ? 32u - __clz(n - 1) : 0u;  // point-index bits
  const bool packed = c.sort_buf && kb + ib <= 64;
  const uint64_t* K = nullptr;  // 64-bit path: sorted keys
  const uint32_t* P = nullptr;  //              sorted original indices
  const uint64_t* W = nullptr;  // packed path: sorted (key << ib | index)
  for (uint32_t i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {  // U points in flight
    float v[U][3];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * blockDim.x;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) v[u][ax] = i < n ? d[3 * i + ax] : o[ax];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * blockDim.x;
      if (i >= n) break;
      uint64_t kk[3];
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) kk[ax] = (uint64_t)floorf(__fdiv_rn(__fsub_rn(v[u][ax], o[ax]), op.voxel));
      const uint64_t key = kk[0] | (kk[1] << bx[0]) | (kk[2] << (bx[0] + bx[1]));
      if (packed) {
        c.key[0][i] = (key << ib) | i;
      } else {
        c.key[0][i] = key;
        idx[i] = i;
      }
    }
  }
  __syncthreads();
  vmark(1);  // key pass
  if (packed) {
    const int r = radix_sort8<U>(c.key[0], c.key[1], n, ib, ib + kb, c.sort_buf);
    W = c.key[r];
  } else {
    const int r = radix_sort(c.key[0], idx, c.key[1], idx2, n, kb, S);
    K = c.key[r];
    P = r ? idx2 : idx;
  }
  const uint64_t imask = ib ? ((1ull << ib) - 1) : 0ull;
  auto key_at = [&](uint32_t k) -> uint64_t { return packed ? W[k] >> ib : K[k]; };
  auto pt_at = [&](uint32_t k) -> uint32_t { return packed ? (uint32_t)(W[k] & imask) : P[k]; };
  vmark(2);  // sort
  // voxel starts (key changes), warp-partitioned: each warp counts the starts
  // in its contiguous chunk, one prefix over the warp totals, then each warp
  // writes its starts in order (two barriers instead of a block scan per tile)
  uint32_t* seg = reinterpret_cast<uint32_t*>(c.ix[2]);
  uint32_t V = 0;
  {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t per = ((n + nw - 1) / nw + 31) & ~31u;
    const uint32_t c0 = min(w * per, n), c1 = min(c0 + per, n);
    auto starts = [&](uint32_t i0, uint32_t (&bal)[U]) {
      bool f[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + 32 * u + lane;
        f[u] = i < c1 && (i == 0 || key_at(i) != key_at(i - 1));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) bal[u] = __ballot_sync(0xffffffffu, f[u]);
    };
    uint32_t cnt = 0;
    for (uint32_t i0 = c0; i0 < c1; i0 += 32 * U) {
      uint32_t bal[U];
      starts(i0, bal);
#pragma unroll
      for (int u = 0; u < U; ++u) cnt += __popc(bal[u]);
    }
    uint32_t* wt = reinterpret_cast<uint32_t*>(S.red);
    __syncthreads();
    if (lane == 0) wt[w] = cnt;
    __syncthreads();
    uint32_t run = 0;
    for (uint32_t k = 0; k < nw; ++k) {
      if (k < w) run += wt[k];
      V += wt[k];
    }
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t i0 = c0; i0 < c1; i0 += 32 * U) {
      uint32_t bal[U];
      starts(i0, bal);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if ((bal[u] >> lane) & 1u) seg[run + __popc(bal[u] & lt)] = i0 + 32 * u + lane;
        run += __popc(bal[u]);
      }
    }
    __syncthreads();
  }
  vmark(3);  // segments
  // 1) gather every moved field into sorted order (alt), one point per thread:
  //    independent loads, many in flight (the per-voxel loop below would
  //    otherwise chain index load -> data load -> add per point)
  //    (4 points per thread per round for 4- and 12-byte points)
  for (int f = 0; f < a.n_bytes_fields; ++f) {
    if (!((mm >> f) & 1u)) continue;
    const uint32_t es = c.elem[f];
    if (es == 12 || es == 4) {
      const uint32_t w = es >> 2;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(c.cur[f]);
      uint32_t* dst = reinterpret_cast<uint32_t*>(c.alt[f]);
      for (uint32_t k0 = threadIdx.x; k0 < n; k0 += 4 * blockDim.x) {
        uint64_t p[4];
        uint32_t v[4][3];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t k = k0 + u * blockDim.x;
          p[u] = k < n ? pt_at(k) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t k = k0 + u * blockDim.x;
          if (k < n) {
            v[u][0] = src[p[u] * w];
            if (w == 3) {
              v[u][1] = src[p[u] * 3 + 1];
              v[u][2] = src[p[u] * 3 + 2];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t k = k0 + u * blockDim.x;
          if (k < n) {
            dst[(uint64_t)k * w] = v[u][0];
            if (w == 3) {
              dst[(uint64_t)k * 3 + 1] = v[u][1];
              dst[(uint64_t)k * 3 + 2] = v[u][2];
            }
          }
        }
      }
    } else {
      for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
        const uint64_t p = pt_at(k);
        if ((es & 3u) == 0) {
          const uint32_t w = es >> 2;
          const uint32_t* src = reinterpret_cast<const uint32_t*>(c.cur[f]) + p * w;
          uint32_t* dst = reinterpret_cast<uint32_t*>(c.alt[f]) + (uint64_t)k * w;
          for (uint32_t q = 0; q < w; ++q) dst[q] = src[q];
        } else {
          for (uint32_t b = 0; b < es; ++b) c.alt[f][(uint64_t)k * es + b] = c.cur[f][p * es + b];
        }
      }
    }
  }
  __syncthreads();
  // 2) per voxel: sequential double sums over its contiguous run -- the sort
  //    is stable, so run order = original point order (grid_subsample's
  //    accumulation order) -- written back into cur (dead after the gather)
  for (uint32_t v = threadIdx.x; v < V; v += blockDim.x) {
    const uint32_t s0 = seg[v], s1 = v + 1 < V ? seg[v + 1] : n;
    const double cnt = (double)(s1 - s0);
    for (int f = 0; f < a.n_bytes_fields; ++f) {
      if (!((mm >> f) & 1u)) continue;
      const bool avg = f == a.role_data || f == a.role_normal || f == a.role_color ||
                       f == a.role_intensity;
      if (avg) {
        const uint32_t comps = c.elem[f] / 4;
        const float* src = reinterpret_cast<const float*>(c.alt[f]);
        float* dst = reinterpret_cast<float*>(c.cur[f]);
        if (comps <= 4) {
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          for (uint32_t k = s0; k < s1; ++k) {
            const float* e = src + (uint64_t)k * comps;
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q)
              if (q < comps) acc[q] = __dadd_rn(acc[q], (double)e[q]);
          }
#pragma unroll
          for (uint32_t q = 0; q < 4; ++q)
            if (q < comps) dst[(uint64_t)v * comps + q] = __double2float_rn(__ddiv_rn(acc[q], cnt));
        } else {
          for (uint32_t q = 0; q < comps; ++q) {
            double acc = 0.0;
            for (uint32_t k = s0; k < s1; ++k) acc = __dadd_rn(acc, (double)src[(uint64_t)k * comps + q]);
            dst[(uint64_t)v * comps + q] = __double2float_rn(__ddiv_rn(acc, cnt));
          }
        }
      } else {
        const uint32_t es = c.elem[f];
        for (uint32_t b = 0; b < es; ++b) c.cur[f][(uint64_t)v * es + b] = c.alt[f][(uint64_t)s0 * es + b];
      }
    }
    if (c.counts) c.counts[v] = (int32_t)(s1 - s0);
  }
  __syncthreads();
  vmark(4);  // means
  if (threadIdx.x == 0) {
    for (int f = 0; f < a.n_bytes_fields; ++f)
      if ((mm >> f) & 1u) c.n[f] = V;
    if (op.counts) {
      c.has_counts = 1;
      c.n_counts = V;
    }
  }
  __syncthreads();
  return kOk;
}

// Applies the op chain (Pipeline map worker, pipeline.cpp:474-480): seed per
// op = mix_seed(base, epoch, index, op id), or `fixed_seed` for the
// single-op cloud-set API.  fail_op = 1-based failing transform.
// (force-inlined: an outlined call would need the address of the kernel's
// WaveArgs parameter, and ptxas would copy all ~3 KB of it to local memory)
template <int MinBlocks>
__device__ __forceinline__ int32_t run_chain(const WaveArgs& a, Cloud& c, Smem& S, uint32_t sample, uint64_t epoch, uint64_t index,
                             const uint64_t* fixed_seed, int32_t& fail_op, int op_begin, int op_end) {
  int32_t status = kOk;
  const int fd = a.role_data;
  long long t0 = (a.op_cycles && threadIdx.x == 0) ? clock64() : 0;
  for (int k = op_begin; status == kOk && k < op_end; ++k) {
    const OpDesc& op = a.ops[k];
    const Seed seed{fixed_seed ? *fixed_seed : rng::mix_seed(a.base_seed, epoch, index, op.seed_op_id),
                    (a.mt_pre && !fixed_seed && a.rng_slot[k] >= 0)
                        ? a.mt_pre + ((uint64_t)sample * a.n_rng + a.rng_slot[k]) * rng::kN
                        : nullptr};
    if (c.n[fd] == 0) {
      status = kEmptyCloud;
    } else {
      switch (op.kind) {
        case kNormalize: status = op_normalize(a, c, S); break;
        case kTranslate: status = op_translate(a, c, S, seed); break;
        case kJitter: status = op_jitter(a, c, S, seed); break;
        case kRotate: status = op_rotate(a, c, S, op, seed); break;
        case kRandomScale: status = op_scale(a, c, S, seed); break;
        case kFlipYz: status = op_flip(a, c, S, seed); break;
        case kColorAugment: status = op_color(a, c, S, seed); break;
        case kRandomCrop: status = op_random_crop(a, c, S, seed); break;
        case kDownsample: status = op_downsample(a, c, S, op, seed); break;
        case kFps: status = op_fps<MinBlocks>(a, c, S, op); break;
        case kRangeCrop: status = op_range_crop(a, c, S, op); break;
        case kVoxel: status = op_voxel<MinBlocks == 1 ? 8 : 4>(a, c, S, op); break;
        default: status = kUnknownOp; break;
      }
    }
    if (status != kOk) fail_op = k + 1;
    if (a.op_cycles && threadIdx.x == 0) {
      const long long t1 = clock64();
      atomicAdd(a.op_cycles + 1 + k, (unsigned long long)(t1 - t0));
      t0 = t1;
    }
  }
  return status;
}

// Carves the per-CTA buffers: staging, 4 index arrays and
// tracked cur/alt pairs — in shared memory when they fit, else a global slab.
__device__ uint8_t* carve(const WaveArgs& a, uint8_t* work, Cloud& proto);

// Byte capacity of a tracked field's buffer.
__device__ __forceinline__ uint64_t field_bytes(const WaveArgs& a, int f) {
  return (uint64_t)a.cap_points * a.field_cap[f] + 16;
}

// Tracked fields and the synthesized "count" field into the sample's batch
// slots (leader CTA).
__device__ __forceinline__ void write_tracked(const WaveArgs& a, const Cloud& c, uint32_t s, int32_t& status) {
  for (int f = 0; f < a.n_bytes_fields && status == kOk; ++f) {
    const int of = a.bytes_out[f];
    if (!((a.tracked_mask >> f) & 1u) || of < 0) continue;
    const uint64_t nb = c.present >> f & 1u ? (uint64_t)c.n[f] * c.elem[f] : 0;
    if (nb > a.out_stride[of]) {
      status = kOutOfBounds;
      break;
    }
    const uint32_t* s32 = reinterpret_cast<const uint32_t*>(c.cur[f]);
    uint8_t* dst = a.out[of] + (uint64_t)s * a.out_stride[of];
    uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
    for (uint64_t i = threadIdx.x; i < nb / 4; i += blockDim.x) d32[i] = s32[i];
    for (uint64_t i = (nb & ~3ull) + threadIdx.x; i < nb; i += blockDim.x) dst[i] = c.cur[f][i];
    if (threadIdx.x == 0) a.out_len[(uint64_t)of * a.n_samples + s] = nb;
  }
  if (status == kOk && a.count_out >= 0) {  // synthesized "count" field (voxel counts, int32 bytes)
    const int of = a.count_out;
    const uint64_t nb = c.has_counts ? (uint64_t)c.n_counts * 4 : 0;
    if (nb > a.out_stride[of]) {
      status = kOutOfBounds;
    } else {
      int32_t* dst = reinterpret_cast<int32_t*>(a.out[of] + (uint64_t)s * a.out_stride[of]);
      for (uint32_t i = threadIdx.x; i < nb / 4; i += blockDim.x) dst[i] = c.counts[i];
      if (threadIdx.x == 0) a.out_len[(uint64_t)of * a.n_samples + s] = nb;
    }
  }
}

// 16-B aligned copy (chain-split hand-off), whole CTA.
__device__ __forceinline__ void copy16(uint8_t* dst, const uint8_t* src, uint64_t nb) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (uint64_t i = threadIdx.x; i < nb / 16; i += blockDim.x) d4[i] = s4[i];
  for (uint64_t i = (nb & ~15ull) + threadIdx.x; i < nb; i += blockDim.x) dst[i] = src[i];
}

// Chain split: the cloud after the prefix ops, to / from the hand-off slot
// [header: status, present, n[8], elem[8], has_counts, n_counts | fields | counts].
__device__ __forceinline__ void handoff_store(const WaveArgs& a, const Cloud& c, uint8_t* hb) {
  for (int f = 0; f < a.n_bytes_fields; ++f)
    if (((a.tracked_mask >> f) & 1u) && ((c.present >> f) & 1u) && c.cur[f] != hb + a.handoff_off[f])
      copy16(hb + a.handoff_off[f], c.cur[f], (uint64_t)c.n[f] * c.elem[f]);
  if (c.has_counts && reinterpret_cast<uint8_t*>(c.counts) != hb + a.handoff_off[kMaxBytesFields])
    copy16(hb + a.handoff_off[kMaxBytesFields], reinterpret_cast<const uint8_t*>(c.counts),
           (uint64_t)c.n_counts * 4);
  if (threadIdx.x == 0) {
    uint32_t* h = reinterpret_cast<uint32_t*>(hb);
    h[1] = c.present;
    for (int f = 0; f < kMaxBytesFields; ++f) {
      h[2 + f] = c.n[f];
      h[10 + f] = c.elem[f];
    }
    h[18] = (uint32_t)c.has_counts;
    h[19] = c.n_counts;
  }
}

// in_place: the cloud's current buffers ARE the hand-off slot (one CTA per
// cloud owns it; ops write alt buffers / in place as usual), no copy.
__device__ __forceinline__ void handoff_load(const WaveArgs& a, Cloud& c, Smem& S, uint8_t* hb, bool in_place) {
  const uint32_t* h = reinterpret_cast<const uint32_t*>(hb);
  if (threadIdx.x == 0) {
    S.cl = S.proto;
    S.cl.present = h[1];
    for (int f = 0; f < kMaxBytesFields; ++f) {
      S.cl.n[f] = h[2 + f];
      S.cl.elem[f] = h[10 + f];
      if (in_place && ((a.tracked_mask >> f) & 1u)) S.cl.cur[f] = hb + a.handoff_off[f];
    }
    S.cl.has_counts = (int32_t)h[18];
    S.cl.n_counts = h[19];
    if (in_place && a.voxel_scratch) S.cl.counts = reinterpret_cast<int32_t*>(hb + a.handoff_off[kMaxBytesFields]);
  }
  __syncthreads();
  if (in_place) return;
  for (int f = 0; f < a.n_bytes_fields; ++f)
    if (((a.tracked_mask >> f) & 1u) && ((c.present >> f) & 1u))
      copy16(c.cur[f], hb + a.handoff_off[f], (uint64_t)c.n[f] * c.elem[f]);
  if (c.has_counts) copy16(reinterpret_cast<uint8_t*>(c.counts), hb + a.handoff_off[kMaxBytesFields],
                           (uint64_t)c.n_counts * 4);
  __syncthreads();
}

// MinBlocks = 1: up to 128 registers (FPS keeps min-distances in registers);
// MinBlocks = 2: <= 64 registers, two CTAs per SM for global-slab clouds.
template <int MinBlocks>
__global__ void __launch_bounds__(512, MinBlocks) k_cloud(WaveArgs a) {
  extern __shared__ __align__(128) uint8_t dyn[];
  Smem& S = *reinterpret_cast<Smem*>(dyn);
  uint8_t* work = dyn + ((sizeof(Smem) + 127) & ~size_t(127));
  for (int i = threadIdx.x; i < 256; i += blockDim.x) S.crc_tab[i] = crc::table_entry(i);
  if (threadIdx.x == 0) {
    dev::mbar_init(&S.bar, 1);
    dev::fence_mbar_init();
  }
  __syncthreads();

  Cloud proto{};
  uint8_t* staging = carve(a, work, proto);
  if (threadIdx.x == 0) S.proto = proto;
  __syncthreads();
  Cloud& c = S.cl;

  // cluster FPS: the fps_cluster CTAs of a cluster run the same sample (the
  // chain redundantly, FPS split over them); only rank 0 writes results
  const uint32_t CL = a.fps_cluster > 1 ? a.fps_cluster : 1;
  const bool leader = (blockIdx.x % CL) == 0;
  uint32_t phase = 0;
  for (uint32_t s = blockIdx.x / CL; s < a.n_samples; s += gridDim.x / CL) {
    const SampleWork sw = a.samples[s];
    if (a.handoff_in) {
      // chain split, a later launch: the cloud after the earlier ops; a failed
      // earlier stage already wrote the (final) status.  Multi-CTA voxel
      // clouds whose keys did not fit the packed sort (vx fallback) take
      // their decoded input and run the voxel ops here instead.
      uint8_t* hb = a.handoff_in + (uint64_t)s * a.handoff_stride;
      int op0 = a.op_begin;
      if (a.vx_state && a.vx_state[s].fallback) {
        hb = a.handoff_fallback + (uint64_t)s * a.handoff_stride;
        op0 = a.vx_first;
      }
      if (reinterpret_cast<const uint32_t*>(hb)[0] != (uint32_t)kOk) continue;  // uniform
      handoff_load(a, c, S, hb, CL == 1);
      int32_t fail_op = 0;
      int32_t status = run_chain<MinBlocks>(a, c, S, s, sw.epoch, sw.index, nullptr, fail_op, op0, a.op_end);
      uint8_t* ho = a.handoff_out ? a.handoff_out + (uint64_t)s * a.handoff_stride : nullptr;
      if (ho && status == kOk) handoff_store(a, c, ho);
      if (status == kOk && leader && !ho) write_tracked(a, c, s, status);
      if (threadIdx.x == 0 && leader && (!ho || status != kOk)) {
        a.sample_status[s] = status;
        a.sample_op[s] = status == kOk ? -1 : fail_op;
        a.sample_where[s] = 0;
      }
      if (ho && threadIdx.x == 0) reinterpret_cast<uint32_t*>(ho)[0] = (uint32_t)status;
      __syncthreads();
      continue;
    }
    const PageRef pg = a.pages[sw.block_page];
    const ScalarRec rec = a.recs[(uint64_t)a.groups[sw.group].first_rec + sw.row];
    int32_t fail_op = 0;
    const long long tc0 = (a.op_cycles && threadIdx.x == 0) ? clock64() : 0;
    // read_sample checks (format.cpp:741-755)
    const bool range_ok = sw.blob_end <= pg.raw_len && sw.blob_start <= sw.blob_end;
    uint64_t* flen = S.flen;
    uint64_t* foff = S.foff;
    uint8_t* hb = a.handoff_out ? a.handoff_out + (uint64_t)s * a.handoff_stride : nullptr;
    if (threadIdx.x == 0) {
      int32_t st0 = rec.status;
      if (st0 == kOk && !range_ok) st0 = kRangeOutOfBounds;
      if (st0 == kOk && rec.n_lens != (uint32_t)a.n_bytes_fields) st0 = kCorruptPage;
      if (st0 == kOk) {
        uint64_t at = 0;
        for (int f = 0; f < a.n_bytes_fields; ++f) {
          flen[f] = rec.lens[f];
          foff[f] = at;
          if (at + flen[f] > sw.blob_end - sw.blob_start) st0 = kRangeOutOfBounds;
          at += flen[f];
        }
      }
      S.pre_status = st0;
      S.cl = S.proto;
      S.cl.present = 0;
      if (hb && a.op_begin == a.op_end)  // decode-only launch: straight into the hand-off slot
        for (int f = 0; f < kMaxBytesFields; ++f)
          if ((a.tracked_mask >> f) & 1u) S.cl.cur[f] = hb + a.handoff_off[f];
    }
    __syncthreads();
    int32_t status = S.pre_status;
    const bool lz4 = (pg.flags & kFlagOuterLz4) != 0;
    if (!lz4 && pg.pay_len != pg.raw_len && status == kOk) status = kCorruptPage;
    const uint8_t* src = lz4 ? a.raw + pg.raw_dst + sw.blob_start
                             : a.bytes + pg.off + kPageHeaderBytes + sw.blob_start;
    const uint64_t blen = range_ok ? sw.blob_end - sw.blob_start : 0;
    const bool need_bytes = status == kOk || pg.crc_mode == 1;

    // ---- stage the blob with one TMA bulk copy (smem mode) ----------------
    const uint8_t* blob = src;
    if (need_bytes && staging && blen > 0) {
      const uintptr_t g0 = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
      const uintptr_t g1 = (reinterpret_cast<uintptr_t>(src) + blen + 15) & ~uintptr_t(15);
      const uint32_t nbytes = (uint32_t)(g1 - g0);
      dev::fence_proxy_async();
      __syncthreads();
      if (threadIdx.x == 0) {
        dev::mbar_expect_tx(&S.bar, nbytes);
        for (uint32_t o = 0; o < nbytes; o += 65536u)
          dev::bulk_g2s(staging + o, reinterpret_cast<const void*>(g0 + o), min(65536u, nbytes - o),
                        &S.bar);
      }
      dev::mbar_wait(&S.bar, phase);
      phase ^= 1;
      blob = staging + (reinterpret_cast<uintptr_t>(src) - g0);
    }
    // ---- fused payload CRC: this sample's share of its page ---------------
    if (pg.crc_mode == 1 && blen > 0) {
      const uint32_t cc = crc::cta_range(S.crc_tab, c_x2n.v, a.shift_tab, blob, blen,
                                         pg.raw_len - sw.blob_end,
                                         reinterpret_cast<uint32_t*>(S.red));
      if (threadIdx.x == 0 && leader) atomicXor(a.page_crc_acc + sw.block_page, cc);
    }

    // ---- decode fields: XOR-delta per blob field (format.cpp:483-493) -----
    if (status == kOk) {
      const bool delta_page = (pg.flags & kFlagInnerDelta) != 0;
      for (int f = 0; f < a.n_bytes_fields && status == kOk; ++f) {
        const bool delta = delta_page && flen[f] >= 8 && (flen[f] % 4) == 0;
        const int of = a.bytes_out[f];
        if ((a.tracked_mask >> f) & 1u) {
          if (flen[f] + 16 > field_bytes(a, f)) {
            status = kOutOfBounds;
            break;
          }
          decode_bytes<1, MinBlocks == 1 ? 8 : 4>(c.cur[f], blob + foff[f], flen[f], delta, S);
          uint32_t e;
          if (f == a.role_data || f == a.role_normal || f == a.role_color) {
            e = 12;
          } else if (f == a.role_intensity) {
            e = 4;
          } else {  // extra per-point field: bytes per point from "data"
            const uint64_t nd = a.role_data >= 0 ? flen[a.role_data] / 12 : 0;
            e = (nd && flen[f] % nd == 0) ? (uint32_t)(flen[f] / nd) : 0;
          }
          if (threadIdx.x == 0) {
            c.elem[f] = e ? e : 1;
            c.n[f] = e ? (uint32_t)(flen[f] / e) : 0;
            if (flen[f] > 0 || f == a.role_data) c.present |= 1u << f;
          }
        } else if (of >= 0) {
          if (flen[f] > a.out_stride[of]) {
            status = kOutOfBounds;
            break;
          }
          if (leader) {
            decode_bytes<1, MinBlocks == 1 ? 8 : 4>(a.out[of] + (uint64_t)s * a.out_stride[of], blob + foff[f],
                                                 flen[f], delta, S);
            if (threadIdx.x == 0) a.out_len[(uint64_t)of * a.n_samples + s] = flen[f];
          }
        }
      }
    }

    __syncthreads();
    if (a.op_cycles && threadIdx.x == 0) atomicAdd(a.op_cycles, (unsigned long long)(clock64() - tc0));
    // ---- the op chain (Pipeline map worker, pipeline.cpp:474-480) ---------
    if (status == kOk && a.n_ops > 0) {
      const int fd = a.role_data;
      // get_points / maybe_unpack checks (transforms.cpp:19-50)
      if (fd < 0) status = kMissingField;
      else if (flen[fd] % 12) status = kMissingField;
      else if (flen[fd] == 0) status = kEmptyCloud;
      if (status == kOk && a.role_normal >= 0 && flen[a.role_normal] % 12) status = kMissingField;
      if (status == kOk && a.role_color >= 0 && flen[a.role_color] % 12) status = kMissingField;
      if (status != kOk) fail_op = 1;
      if (status == kOk)
        status = run_chain<MinBlocks>(a, c, S, s, sw.epoch, sw.index, nullptr, fail_op, a.op_begin, a.op_end);
    }

    // ---- chain split, first launch: hand the cloud to the next launch -----
    if (hb && status == kOk) handoff_store(a, c, hb);
    // ---- write tracked fields + scalar values into the batch slot --------
    const long long tc2 = (a.op_cycles && threadIdx.x == 0) ? clock64() : 0;
    if (status == kOk && leader) {
      if (!hb) write_tracked(a, c, s, status);
      uint32_t vo = rec.vals_off;
      for (int f = 0; f < a.n_fields && status == kOk; ++f) {
        const FieldDesc fdsc = a.fields[f];
        if (fdsc.kind == kBytes) continue;
        const uint8_t* v = a.vals + vo;
        uint32_t nb, skip = 0;
        if (fdsc.kind == kString) {
          nb = *reinterpret_cast<const uint32_t*>(v);
          v += 4;
          skip = 4;
        } else {
          nb = ((fdsc.kind == kInt64 || fdsc.kind == kFloat64) ? 8u : 4u) * fdsc.elems;
        }
        const int of = fdsc.out_index;
        if (nb > a.out_stride[of]) {
          status = kOutOfBounds;
          break;
        }
        uint8_t* dst = a.out[of] + (uint64_t)s * a.out_stride[of];
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) dst[i] = v[i];
        if (threadIdx.x == 0) a.out_len[(uint64_t)of * a.n_samples + s] = nb;
        vo += nb + skip;
      }
    }
    if (threadIdx.x == 0 && leader && (!hb || status != kOk)) {  // split: the second launch reports success
      a.sample_status[s] = status;
      a.sample_op[s] = status == kOk ? -1 : fail_op;
      a.sample_where[s] = 0;
    }
    if (hb && threadIdx.x == 0) reinterpret_cast<uint32_t*>(hb)[0] = (uint32_t)status;
    if (a.op_cycles && threadIdx.x == 0)
      atomicAdd(a.op_cycles + a.n_ops + 1, (unsigned long long)(clock64() - tc2));
    __syncthreads();
  }
}

__device__ uint8_t* carve(const WaveArgs& a, uint8_t* work, Cloud& proto) {
  uint8_t* gbase = a.gscratch ? a.gscratch + (uint64_t)blockIdx.x * a.gscratch_per_cta : nullptr;
  uint64_t soff = 0, goff = 0;
  uint8_t* ptr[26];
  for (int b = 0; b < 26; ++b) {
    const uint64_t nb = (a.buf_bytes[b] + 127) & ~uint64_t(127);
    if (!nb) {
      ptr[b] = nullptr;
    } else if ((a.buf_smem_mask >> b) & 1u) {
      ptr[b] = work + soff;
      soff += nb;
    } else {
      ptr[b] = gbase + goff;
      goff += nb;
    }
  }
  proto.cap = a.cap_points;
  for (int k = 0; k < 4; ++k) proto.ix[k] = reinterpret_cast<int32_t*>(ptr[1 + k]);
  for (int f = 0; f < kMaxBytesFields; ++f) {
    proto.cur[f] = ptr[5 + f];
    proto.alt[f] = ptr[13 + f];
  }
  proto.key[0] = reinterpret_cast<uint64_t*>(ptr[21]);
  proto.key[1] = reinterpret_cast<uint64_t*>(ptr[22]);
  proto.counts = reinterpret_cast<int32_t*>(ptr[23]);
  proto.fps_buf = ptr[24];
  proto.sort_buf = reinterpret_cast<uint32_t*>(ptr[25]);
  return ptr[0];  // TMA staging buffer (shared) or nullptr
}

// pcp_apply_map: one op over a CSR cloud set (apply_map per cloud with an
// explicit seed, transforms.hpp:33-34).
__global__ void __launch_bounds__(512, 1) k_apply_set(WaveArgs a) {
  extern __shared__ __align__(128) uint8_t dyn[];
  Smem& S = *reinterpret_cast<Smem*>(dyn);
  uint8_t* work = dyn + ((sizeof(Smem) + 127) & ~size_t(127));
  Cloud proto{};
  carve(a, work, proto);
  if (threadIdx.x == 0) S.proto = proto;
  __syncthreads();
  Cloud& c = S.cl;
  const uint32_t CL = a.fps_cluster > 1 ? a.fps_cluster : 1;
  const bool leader = (blockIdx.x % CL) == 0;
  for (uint32_t s = blockIdx.x / CL; s < a.n_samples; s += gridDim.x / CL) {
    const uint64_t p0 = a.set_offset[s], p1 = a.set_offset[s + 1];
    const uint64_t n = p1 >= p0 ? p1 - p0 : 0;
    if (threadIdx.x == 0) {
      S.cl = S.proto;
      S.cl.present = 0;
    }
    __syncthreads();
    int32_t status = kOk, fail_op = 0;
    if (n > a.cap_points) status = kOutOfBounds;
    for (int f = 0; status == kOk && f < a.n_bytes_fields; ++f) {
      if (!((a.tracked_mask >> f) & 1u)) continue;
      const uint32_t e = a.set_elem[f];
      const uint8_t* src = a.set_src[f] + p0 * e;
      const uint64_t nb = n * e;
      if ((e & 3) == 0) {
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
        uint32_t* d32 = reinterpret_cast<uint32_t*>(c.cur[f]);
        for (uint64_t i = threadIdx.x; i < nb / 4; i += blockDim.x) d32[i] = s32[i];
      } else {
        for (uint64_t i = threadIdx.x; i < nb; i += blockDim.x) c.cur[f][i] = src[i];
      }
      if (threadIdx.x == 0) {
        c.n[f] = (uint32_t)n;
        c.elem[f] = e;
        if (n > 0 || f == a.role_data) c.present |= 1u << f;
      }
    }
    __syncthreads();
    if (status == kOk && n == 0) status = kEmptyCloud;
    if (status == kOk) status = run_chain<1>(a, c, S, s, 0, 0, a.set_seeds + s, fail_op, 0, a.n_ops);
    if (status == kOk && leader) {
      for (int f = 0; f < a.n_bytes_fields && status == kOk; ++f) {
        if (!((a.tracked_mask >> f) & 1u) || !a.set_out[f]) continue;
        const uint64_t nb = (uint64_t)c.n[f] * c.elem[f];
        if (c.n[f] > a.set_out_cap) {
          status = kOutOfBounds;
          break;
        }
        uint8_t* dst = a.set_out[f] + (uint64_t)s * a.set_out_cap * a.set_elem[f];
        for (uint64_t i = threadIdx.x; i < nb; i += blockDim.x) dst[i] = c.cur[f][i];
      }
    }
    if (status == kOk && leader && a.set_voxel_count && c.has_counts)
      for (uint32_t i = threadIdx.x; i < c.n_counts && i < a.set_out_cap; i += blockDim.x)
        a.set_voxel_count[(uint64_t)s * a.set_out_cap + i] = c.counts[i];
    if (threadIdx.x == 0 && leader) {
      a.sample_status[s] = status;
      if (a.set_count) a.set_count[s] = status == kOk ? c.n[a.role_data] : 0;
    }
    __syncthreads();
  }
}

// pcp_crc32_ranges: one CTA per range.
__global__ void k_crc_ranges(const uint8_t* bytes, const uint64_t* off, const uint64_t* len,
                             uint32_t n, const uint32_t* shift_tab, uint32_t* out) {
  __shared__ uint32_t tab[256];
  __shared__ uint32_t red[32];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = crc::table_entry(i);
  __syncthreads();
  for (uint32_t r = blockIdx.x; r < n; r += gridDim.x) {
    const uint32_t c = crc::cta_range(tab, c_x2n.v, shift_tab, bytes + off[r], len[r], 0, red);
    if (threadIdx.x == 0) out[r] = c;
  }
}

// pcp_decode_pages: one CTA per serialized page — header, CRC, LZ4 or raw,
// then the inner XOR-delta columns (decode_block_page, format.cpp:243-266).
__global__ void k_decode_pages(const uint8_t* bytes, const uint64_t* page_off, uint32_t n_pages,
                               uint8_t* out, const uint64_t* out_off, const uint32_t* col_first,
                               const uint64_t* col_off, const uint64_t* col_len,
                               const uint32_t* shift_tab, const uint64_t* scratch_off,
                               uint8_t* scratch, int32_t* status) {
  __shared__ uint32_t tab[256];
  __shared__ uint32_t red[32];
  __shared__ __align__(16) uint32_t ctl[lz4p::kSmemWords];
  __shared__ Lz4Seq seqs[32];
  __shared__ int32_t sst;
  __shared__ uint32_t scount;
  __shared__ int32_t st_sh;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = crc::table_entry(i);
  __syncthreads();
  for (uint32_t pi = blockIdx.x; pi < n_pages; pi += gridDim.x) {
    const uint8_t* pg = bytes + page_off[pi];
    uint8_t flags = pg[0];
    uint64_t raw_len = 0, pay_len = 0;
    uint32_t crc_stored = 0;
    for (int b = 0; b < 8; ++b) raw_len |= (uint64_t)pg[1 + b] << (8 * b);
    for (int b = 0; b < 8; ++b) pay_len |= (uint64_t)pg[9 + b] << (8 * b);
    for (int b = 0; b < 4; ++b) crc_stored |= (uint32_t)pg[17 + b] << (8 * b);
    const uint8_t* pay = pg + kPageHeaderBytes;
    uint8_t* dst = out + out_off[pi];
    const uint32_t c = crc::cta_range(tab, c_x2n.v, shift_tab, pay, pay_len, 0, red);
    if (threadIdx.x == 0) st_sh = (c == crc_stored) ? kOk : kChecksumMismatch;
    __syncthreads();
    if (st_sh == kOk) {
      if (flags & kFlagOuterLz4) {
        int32_t r = kCorruptPage;
        if (pay_len < 0xFFFFFFF0ull && raw_len < 0xFFFFFFF0ull) {
          const lz4p::Scratch sc = lz4p::carve_scratch(scratch + scratch_off[pi], pay_len);
          r = lz4p::decode_block(pay, (uint32_t)pay_len, dst, (uint32_t)raw_len, sc, ctl);
          if (r < 0) {
            if (threadIdx.x < 32) {
              const int32_t q = warp_lz4_decode(pay, pay_len, dst, raw_len, seqs, &sst, &scount);
              if (threadIdx.x == 0) ctl[5] = (uint32_t)q;
            }
            __syncthreads();
            r = (int32_t)ctl[5];
          }
        }
        if (threadIdx.x == 0) st_sh = r;
      } else if (flags & kFlagStoredRaw) {
        if (pay_len != raw_len) {
          if (threadIdx.x == 0) st_sh = kCorruptPage;
        } else {
          for (uint64_t i = threadIdx.x; i < raw_len; i += blockDim.x) dst[i] = pay[i];
        }
      } else if (threadIdx.x == 0) {
        st_sh = kCorruptPage;
      }
    }
    __syncthreads();
    if (st_sh == kOk && (flags & kFlagInnerDelta)) {
      const uint32_t c0 = col_first[pi], c1 = col_first[pi + 1];
      if (threadIdx.x == 0)
        for (uint32_t k = c0; k < c1; ++k) {
          if (col_off[k] + col_len[k] > raw_len) { st_sh = kColumnOutOfRange; break; }
          if (col_len[k] % 4) { st_sh = kBadAlignment; break; }
        }
      __syncthreads();
      // one warp per column, 32-word chunks, byte-addressed (any alignment)
      const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      if (st_sh == kOk)
        for (uint32_t k = c0 + wid; k < c1; k += nw) {
          uint8_t* col = dst + col_off[k];
          const uint64_t nwd = col_len[k] / 4;
          uint32_t carry = 0;
          for (uint64_t base = 0; base < nwd; base += 32) {
            const uint64_t i = base + lane;
            uint32_t v = 0;
            if (i < nwd)
              v = (uint32_t)col[4 * i] | ((uint32_t)col[4 * i + 1] << 8) |
                  ((uint32_t)col[4 * i + 2] << 16) | ((uint32_t)col[4 * i + 3] << 24);
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
              if ((int)lane >= o) v ^= y;
            }
            v ^= carry;
            __syncwarp();
            if (i < nwd) {
              col[4 * i] = (uint8_t)v;
              col[4 * i + 1] = (uint8_t)(v >> 8);
              col[4 * i + 2] = (uint8_t)(v >> 16);
              col[4 * i + 3] = (uint8_t)(v >> 24);
            }
            carry = __shfl_sync(0xffffffffu, v, 31);
            __syncwarp();
          }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) status[pi] = st_sh;
    __syncthreads();
  }
}

// Page CRC verdicts, then the per-sample status in read_sample order:
// scalar page, block page, record, ops (format.cpp:687-757).
__global__ void k_finalize(WaveArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.n_pages) {
    const PageRef pg = a.pages[i];
    if (a.page_status[i] == kOk && a.page_crc_acc[i] != pg.crc) a.page_status[i] = kChecksumMismatch;
  }
}

__global__ void k_sample_status(WaveArgs a) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n_samples) return;
  const SampleWork sw = a.samples[s];
  const int32_t sp = a.page_status[sw.scalar_page];
  const int32_t bp = a.page_status[sw.block_page];
  if (sp != kOk) {
    a.sample_status[s] = sp;
    a.sample_op[s] = 0;
    a.sample_where[s] = 1;
  } else if (bp != kOk) {
    a.sample_status[s] = bp;
    a.sample_op[s] = 0;
    a.sample_where[s] = 2;
  }
}

// =========================================================================
// launch wrappers
// =========================================================================
void upload_x2n(cudaStream_t st) {
  static bool done = false;
  if (done) return;
  const crc::X2N t = crc::make_x2n();
  cudaMemcpyToSymbolAsync(c_x2n, &t, sizeof(t), 0, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
  done = true;
}

void build_shift_table(uint32_t* h_tab) {
  const crc::X2N t = crc::make_x2n();
  // x^(8*256*k): repeated multiplication by x^(8*256) = x^(2^11)
  const uint32_t step = t.v[11];
  uint32_t p = 1u << 31;
  for (uint32_t k = 0; k < crc::kShiftEntries; ++k) {
    h_tab[k] = p;
    p = crc::multmodp(step, p);
  }
  // byte-sliced multiplication tables by x^(8 * kChunk * stride)
  for (int i = 0; i < 3; ++i) {
    const uint32_t S = h_tab[crc::kMulStrides[i]];
    uint32_t* T = h_tab + crc::kShiftEntries + 1024 * i;
    for (uint32_t b = 0; b < 4; ++b)
      for (uint32_t v = 0; v < 256; ++v) T[256 * b + v] = crc::multmodp(S, v << (8 * b));
  }
}

uint64_t lz4_scratch_bytes(uint64_t pay) { return lz4p::scratch_bytes(pay); }

size_t cloud_smem_fixed() { return (sizeof(Smem) + 127) & ~size_t(127); }

cudaError_t launch_crc_windows(const uint8_t* bytes, const CrcWindow* win, uint32_t n_win,
                               const uint32_t* shift_tab, uint32_t* acc, int sms,
                               cudaStream_t st) {
  if (!n_win) return cudaSuccess;
  const uint32_t warps = 8;
  uint32_t grid = (n_win + warps - 1) / warps;
  grid = grid > (uint32_t)sms * 8 ? (uint32_t)sms * 8 : grid;
  k_crc_windows<<<grid, warps * 32, 0, st>>>(bytes, win, n_win, shift_tab, acc);
  return cudaGetLastError();
}

cudaError_t launch_page_decode(const uint8_t* bytes, uint8_t* raw, const PageRef* pages,
                               const uint32_t* todo, const uint64_t* scratch_off,
                               uint8_t* scratch, uint32_t n_todo, int32_t* status,
                               cudaStream_t st, long long* timing, uint32_t* pj_ptr,
                               uint32_t* pj_changed, uint32_t pj_rounds, uint8_t* pj_flags,
                               uint32_t pj_split) {
  if (!n_todo) return cudaSuccess;
  static bool carve = [] {  // static shared memory only: ask for the max carveout
    cudaFuncSetAttribute(k_page_decode, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return true;
  }();
  (void)carve;
  k_page_decode<<<n_todo, kDecodeThreads, 0, st>>>(bytes, raw, pages, todo, scratch_off, scratch, n_todo,
                                        status, timing);
  static const uint32_t match_threads = [] {  // PCP_MATCH_THREADS: sweep switch (32..kMatchThreads)
    const char* e = std::getenv("PCP_MATCH_THREADS");
    const int v = e ? std::atoi(e) : (int)kMatchThreads;
    return (uint32_t)std::max(32, std::min((int)kMatchThreads, v / 32 * 32));
  }();
  if (pj_ptr) {  // phase 4 by page-wide pointer jumping
    const dim3 g(n_todo, pj_split);  // CTAs per page: ~64 KB of the largest page each, <= kPjSplit
    k_pj_init<<<g, 256, 0, st>>>(raw, pages, todo, scratch_off, scratch, pj_ptr, pj_flags);
    k_pj_matches<<<g, 256, 0, st>>>(raw, pages, todo, scratch_off, scratch, pj_ptr, pj_flags);
    cudaMemsetAsync(pj_changed, 0, 4ull * pj_rounds * n_todo, st);
    for (uint32_t r = 0; r < pj_rounds; ++r)
      k_pj_round<<<g, 256, 0, st>>>(raw, pages, todo, scratch_off, scratch, pj_ptr, pj_flags, pj_changed,
                                   n_todo, r);
    k_pj_gather<<<g, 256, 0, st>>>(raw, pages, todo, scratch_off, scratch, pj_ptr, pj_flags);
    return cudaGetLastError();
  }
  k_page_matches<<<n_todo, match_threads, 0, st>>>(raw, pages, todo, scratch_off, scratch, n_todo, timing);
  return cudaGetLastError();
}

namespace {
template <typename K>
cudaError_t launch_clustered(K kern, const WaveArgs& a, int grid, int threads, size_t smem,
                             cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.fps_cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}
}  // namespace

// MT19937-64 seeding for every (sample, RNG op) of the wave, one thread
// each: the 311-step serial recurrence (std::mt19937_64::seed) leaves
// k_cloud's critical path, where thread 0 ran it while the CTA waited (~8 K
// cycles per downsample and ~4 K per first_draws op).  Op order: rng_slot.
// Ops that take only their first few engine outputs (first_draws) get those
// outputs, tempered, instead of the 312-word state: the recurrence stops at
// word kM + k and 8 k bytes are written instead of 2.5 KB.  Full states
// (jitter, colour augment, downsample) are written 32 B per store, so every
// lane fills whole sectors.
__device__ __forceinline__ int first_draw_count(int kind) {
  switch (kind) {
    case kTranslate: return 3;
    case kRandomCrop: return 6;
    case kRotate:
    case kRandomScale:
    case kFlipYz: return 1;
    default: return 0;  // full state
  }
}

__global__ void __launch_bounds__(64) k_seed_states(WaveArgs a) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (uint64_t)a.n_samples * a.n_rng) return;
  const uint32_t s = (uint32_t)(t / a.n_rng), j = (uint32_t)(t % a.n_rng);
  int k = 0;
  while (k < a.n_ops && a.rng_slot[k] != (int8_t)j) ++k;
  const SampleWork sw = a.samples[s];
  uint64_t x = rng::mix_seed(a.base_seed, sw.epoch, sw.index, a.ops[k].seed_op_id);
  uint64_t* out = a.mt_pre + t * rng::kN;
  const int nd = first_draw_count(a.ops[k].kind);
  if (nd > 0) {
    uint64_t lo[9], hi[8];  // words 0..nd and kM..kM+nd-1
    lo[0] = x;
    for (uint32_t i = 1; i < (uint32_t)rng::kM + nd; ++i) {
      x = rng::seed_step(x, i);
      if (i <= (uint32_t)nd) lo[i] = x;
      if (i >= (uint32_t)rng::kM) hi[i - rng::kM] = x;
    }
    for (int i = 0; i < nd; ++i) out[i] = rng::temper(rng::twist_word(lo[i], lo[i + 1], hi[i]));
    return;
  }
  uint64_t w4[4];
  w4[0] = x;
  for (uint32_t i = 1; i < (uint32_t)rng::kN; ++i) {
    x = rng::seed_step(x, i);
    w4[i & 3] = x;
    if ((i & 3) == 3) {
      uint4* o = reinterpret_cast<uint4*>(out + i - 3);
      o[0] = make_uint4((uint32_t)w4[0], (uint32_t)(w4[0] >> 32), (uint32_t)w4[1], (uint32_t)(w4[1] >> 32));
      o[1] = make_uint4((uint32_t)w4[2], (uint32_t)(w4[2] >> 32), (uint32_t)w4[3], (uint32_t)(w4[3] >> 32));
    }
  }
}

cudaError_t launch_wave(const WaveArgs& a, int grid, int grid_pre, int threads, size_t smem,
                        cudaStream_t st, cudaEvent_t k0, cudaEvent_t k1, const VxArgs* vx,
                        uint32_t vx_tiles, uint32_t vx_btiles, int sms, cudaEvent_t v0, cudaEvent_t v1,
                        uint8_t* handoff_a) {
  if (a.n_groups) k_scalar_parse<<<(a.n_groups + 127) / 128, 128, 0, st>>>(a);
  if (a.mt_pre && a.n_samples && a.n_rng) {
    const uint64_t n = (uint64_t)a.n_samples * a.n_rng;
    k_seed_states<<<(uint32_t)((n + 63) / 64), 64, 0, st>>>(a);
  }
  if (k0) cudaEventRecord(k0, st);
  auto one_cta_per_cloud = [&](const WaveArgs& x, int g) {
    if (x.min_blocks == 2) k_cloud<2><<<g, threads, smem, st>>>(x);
    else k_cloud<1><<<g, threads, smem, st>>>(x);
  };
  if (a.n_samples) {
    if (vx) {
      // decode-only launch into the hand-off slots A, the multi-CTA voxel
      // stage (A voxelized in place, B scratch), then the rest of the chain
      // from A (with a cluster FPS split: the ops before the FPS write A back)
      const int g1 = a.fps_cluster > 1 ? grid_pre : grid;
      WaveArgs l1 = a;
      l1.fps_cluster = 1;
      l1.op_begin = 0;
      l1.op_end = a.vx_first;
      l1.handoff_in = nullptr;
      l1.handoff_out = handoff_a;
      l1.vx_state = nullptr;
      one_cta_per_cloud(l1, g1);
      if (v0) cudaEventRecord(v0, st);
      cudaError_t e = launch_voxel_wave(*vx, vx_tiles, vx_btiles, sms, st);
      if (e != cudaSuccess) return e;
      if (v1) cudaEventRecord(v1, st);
      const int stop = a.split_at ? a.split_at : a.n_ops;
      const bool l2_runs = !a.split_at || a.vx_last + 1 < stop;
      if (l2_runs) {
        WaveArgs l2 = a;
        l2.fps_cluster = 1;
        l2.op_begin = a.vx_last + 1;
        l2.op_end = stop;
        l2.handoff_in = handoff_a;
        l2.handoff_out = a.split_at ? handoff_a : nullptr;
        one_cta_per_cloud(l2, g1);
      }
      if (a.split_at) {
        WaveArgs l3 = a;
        l3.op_begin = a.split_at;
        l3.op_end = a.n_ops;
        l3.handoff_in = handoff_a;
        l3.handoff_out = nullptr;
        if (l2_runs) l3.vx_state = nullptr;
        e = launch_clustered(k_cloud<1>, l3, grid, threads, smem, st);
        if (e != cudaSuccess) return e;
      }
    } else if (a.fps_cluster > 1 && a.split_at > 0) {
      // chain split: ops [0, split_at) one CTA per cloud, then the cluster
      WaveArgs pre = a, post = a;
      pre.fps_cluster = 1;
      pre.op_begin = 0;
      pre.op_end = a.split_at;
      pre.handoff_in = nullptr;
      pre.handoff_out = handoff_a;
      post.op_begin = a.split_at;
      post.op_end = a.n_ops;
      post.handoff_in = handoff_a;
      post.handoff_out = nullptr;
      k_cloud<1><<<grid_pre, threads, smem, st>>>(pre);
      const cudaError_t e = launch_clustered(k_cloud<1>, post, grid, threads, smem, st);
      if (e != cudaSuccess) return e;
    } else if (a.fps_cluster > 1) {
      const cudaError_t e = launch_clustered(k_cloud<1>, a, grid, threads, smem, st);
      if (e != cudaSuccess) return e;
    } else {
      one_cta_per_cloud(a, grid);
    }
  }
  if (k1) cudaEventRecord(k1, st);
  if (a.n_pages) k_finalize<<<(a.n_pages + 255) / 256, 256, 0, st>>>(a);
  if (a.n_samples) k_sample_status<<<(a.n_samples + 255) / 256, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Per-wave CSR of the variable-length batch fields (Batch::stacked order,
// pipeline.cpp:170-200).  k_wave_offsets: one CTA per batch field scans the
// wave's out_len into sample byte offsets (varlen fields) and flags fields
// whose samples all fill their slot exactly ("dense": the slots are then
// already contiguous and stay in place).  k_compact_wave: every (varlen
// field, sample) pair of a non-dense field copies its bytes from its slot to
// compact + offset.  Two launches per wave replace a compaction launch and a
// stream sync per batch per field.
__global__ void __launch_bounds__(1024) k_wave_offsets(const uint64_t* __restrict__ out_len, WaveCsr c,
                                                       uint32_t n) {
  const uint32_t f = blockIdx.x;
  __shared__ uint64_t warp_sum[32];
  __shared__ uint64_t carry;
  __shared__ int all_dense;
  if (threadIdx.x == 0) {
    carry = 0;
    all_dense = 1;
  }
  __syncthreads();
  const int vi = c.var_index[f];
  uint64_t* woff = vi >= 0 ? c.woff + (uint64_t)vi * (n + 1) : nullptr;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bool dense = true;
  for (uint32_t base = 0; base < n; base += blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    const uint64_t L = s < n ? out_len[(uint64_t)f * n + s] : 0;
    if (s < n && L != c.stride[f]) dense = false;
    if (!woff) continue;
    uint64_t v = L;  // inclusive warp scan
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= (uint32_t)d) v += y;
    }
    if (lane == 31) warp_sum[warp] = v;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = lane < (blockDim.x >> 5) ? warp_sum[lane] : 0;
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= (uint32_t)d) w += y;
      }
      warp_sum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const uint64_t excl = carry + (warp ? warp_sum[warp - 1] : 0) + v - L;
    if (s < n) woff[s] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + L;
    __syncthreads();
  }
  if (!dense) atomicAnd(&all_dense, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    c.dense[f] = (uint32_t)all_dense;
    if (woff) woff[n] = carry;
  }
}

__global__ void k_compact_wave(const uint64_t* __restrict__ out_len, WaveCsr c, uint32_t n) {
  const uint64_t items = (uint64_t)c.n_var * n;
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const uint32_t vi = (uint32_t)(it / n), s = (uint32_t)(it % n);
    const int f = c.var_field[vi];
    if (c.dense[f]) continue;  // uniform per CTA
    const uint64_t L = out_len[(uint64_t)f * n + s];
    const uint8_t* src = c.outs[f] + (uint64_t)s * c.stride[f];
    uint8_t* dst = c.compact[f] + c.woff[(uint64_t)vi * (n + 1) + s];
    if ((((uintptr_t)src | (uintptr_t)dst) & 15u) == 0) {
      const uint4* s16 = reinterpret_cast<const uint4*>(src);
      uint4* d16 = reinterpret_cast<uint4*>(dst);
      for (uint64_t k = threadIdx.x; k < L / 16; k += blockDim.x) d16[k] = s16[k];
      for (uint64_t k = (L & ~15ull) + threadIdx.x; k < L; k += blockDim.x) dst[k] = src[k];
    } else if ((((uintptr_t)src | (uintptr_t)dst) & 3u) == 0) {
      const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
      uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
      for (uint64_t k = threadIdx.x; k < L / 4; k += blockDim.x) d4[k] = s4[k];
      for (uint64_t k = (L & ~3ull) + threadIdx.x; k < L; k += blockDim.x) dst[k] = src[k];
    } else {
      for (uint64_t k = threadIdx.x; k < L; k += blockDim.x) dst[k] = src[k];
    }
  }
}

cudaError_t launch_wave_csr(const uint64_t* out_len, const WaveCsr& c, uint32_t n, int sms,
                            cudaStream_t st) {
  if (!n || !c.n_out) return cudaSuccess;
  k_wave_offsets<<<c.n_out, 1024, 0, st>>>(out_len, c, n);
  if (c.n_var) {
    const uint64_t items = (uint64_t)c.n_var * n;
    const uint32_t grid = (uint32_t)std::min<uint64_t>(items, (uint64_t)sms * 8);
    k_compact_wave<<<grid, 256, 0, st>>>(out_len, c, n);
  }
  return cudaGetLastError();
}

// Wave results (status / op / where / lengths) stored straight into mapped
// pinned host memory by the SMs: posted PCIe writes, so the small result
// read-back never queues in the copy engine behind (or ahead of) the bulk
// batch copies of other waves.  n is a multiple of 16, both ends 16-B aligned.
__global__ void k_store_host(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t n16) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

cudaError_t launch_store_host(const uint8_t* src, uint8_t* dst_mapped, uint64_t n, cudaStream_t st) {
  const uint64_t n16 = (n + 15) / 16;
  if (!n16) return cudaSuccess;
  const uint32_t blocks = (uint32_t)std::min<uint64_t>(148, (n16 + 255) / 256);
  k_store_host<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst_mapped), n16);
  return cudaGetLastError();
}

cudaError_t occupancy_cloud(int* n, int threads, size_t smem, int min_blocks) {
  return min_blocks == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, k_cloud<2>, threads, smem)
                         : cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, k_cloud<1>, threads, smem);
}

cudaError_t launch_apply_set(const WaveArgs& a, int grid, int threads, size_t smem,
                             cudaStream_t st) {
  cudaError_t e = set_apply_smem(smem);
  if (e != cudaSuccess) return e;
  if (!a.n_samples) return cudaSuccess;
  if (a.fps_cluster > 1) return launch_clustered(k_apply_set, a, grid, threads, smem, st);
  k_apply_set<<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_crc_ranges(const uint8_t* bytes, const uint64_t* off, const uint64_t* len,
                              uint32_t n, const uint32_t* shift_tab, uint32_t* out,
                              cudaStream_t st) {
  if (!n) return cudaSuccess;
  k_crc_ranges<<<n < 4096 ? n : 4096, 256, 0, st>>>(bytes, off, len, n, shift_tab, out);
  return cudaGetLastError();
}

cudaError_t launch_decode_pages(const uint8_t* bytes, const uint64_t* page_off, uint32_t n,
                                uint8_t* out, const uint64_t* out_off, const uint32_t* col_first,
                                const uint64_t* col_off, const uint64_t* col_len,
                                const uint32_t* shift_tab, const uint64_t* scratch_off,
                                uint8_t* scratch, int32_t* status, cudaStream_t st) {
  if (!n) return cudaSuccess;
  k_decode_pages<<<n < 4096 ? n : 4096, 256, 0, st>>>(bytes, page_off, n, out, out_off, col_first,
                                                     col_off, col_len, shift_tab, scratch_off,
                                                     scratch, status);
  return cudaGetLastError();
}

cudaError_t set_apply_smem(size_t bytes) {
  return cudaFuncSetAttribute(k_apply_set, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}


cudaError_t occupancy_cloud_clusters(int* n, int threads, size_t smem, uint32_t cluster, bool apply) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cluster * 64);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return apply ? cudaOccupancyMaxActiveClusters(n, k_apply_set, &cfg)
               : cudaOccupancyMaxActiveClusters(n, k_cloud<1>, &cfg);
}

cudaError_t set_cloud_smem(size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(k_cloud<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_cloud<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace pcp
