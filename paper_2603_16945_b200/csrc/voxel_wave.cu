// voxel_wave.cu — multi-CTA voxel / grid subsample (App. C)
// for large clouds, with an optional leading range crop.
//
// k_cloud runs one CTA per cloud; a 1 M-point S3DIS room then sorts its
// keys in a per-CTA global slab, and with ~300 rooms in flight those slabs
// never fit in L2 (round 1: 23.6x the algorithmic DRAM traffic).  Here every
// cloud of a wave is spread over many CTAs in tiles of kTile points, and
// each stage is one launch over all tiles of the wave:
//
//   prep      one CTA: per-cloud tile ranges, statuses from the decoded slot
//   bounds    per tile: range-crop mask, kept count, min/max/NaN per axis
//   plan      per cloud: compaction offsets of the kept points, origin, key
//             widths (per-axis key minus its minimum: order-preserving),
//             App. C range checks -> status, or "fallback" when the packed
//             word does not fit 64 bits
//   keys      per tile: word = key << ib | point index for kept points,
//             compacted in point order; digit histograms of every pass
//   3 x pass  LSD radix sort over 8-bit digits, reduce-then-scan:
//             upsweep (tile digit counts) / colscan (per digit, over tiles)
//             / downsweep (stable in-tile ranks, scatter)
//   segs      per tile: voxel starts (key changes) counted, scanned per cloud
//   gather    payload of the moved fields into sorted order (A -> B)
//   means     one thread per voxel: count, sequential double sums over its
//             run in point order (the sort is stable) = bit-exact App. C
//             means, first point of gathered extra fields (B -> A)
//   finish    per cloud: the hand-off header (A) the rest of the chain reads
//
// The words carry the point index, so (key, index) order is the App. C
// order (ascending key, original order inside a voxel) and the means sum in
// exactly the sequence op_voxel (kernels.cu) and the restatement use.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_util.cuh"
#include "voxel_wave.h"

namespace pcp {
namespace {

constexpr uint32_t kThreads = 256;
constexpr uint32_t kItems = 8;
constexpr uint32_t kTile = kThreads * kItems;  // points / words per tile
constexpr uint32_t kWarps = kThreads / 32;

__device__ __forceinline__ uint32_t ord_f(float x) {  // float order as unsigned order
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__device__ __forceinline__ const uint8_t* slot(const VxArgs& v, const uint8_t* base, uint32_t s) {
  return base + (uint64_t)s * v.stride;
}
__device__ __forceinline__ const uint32_t* hdr(const VxArgs& v, const uint8_t* base, uint32_t s) {
  return reinterpret_cast<const uint32_t*>(slot(v, base, s));
}

// App. C key of one coordinate: k = (int32)floorf((p - o) / v)
__device__ __forceinline__ float qkey(float p, float o, float vs) {
  return floorf(__fdiv_rn(__fsub_rn(p, o), vs));
}

__device__ __forceinline__ bool in_box(const VxArgs& v, float x, float y, float z) {
  return !v.has_crop || (x >= v.lo[0] && x <= v.hi[0] && y >= v.lo[1] && y <= v.hi[1] &&
                         z >= v.lo[2] && z <= v.hi[2]);
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if ((int)lane >= o) x += y;
  }
  return x;
}

// Block-wide exclusive scan of one value per thread (kThreads); returns the
// exclusive prefix, *total = sum.  `sh` >= kWarps + 1 words.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* sh, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t inc = warp_incl_scan(x);
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (uint32_t k = 0; k < kWarps; ++k) {
      const uint32_t c = sh[k];
      sh[k] = acc;
      acc += c;
    }
    sh[kWarps] = acc;
  }
  __syncthreads();
  const uint32_t r = sh[w] + inc - x;
  *total = sh[kWarps];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- prep
__global__ void __launch_bounds__(1024) k_vx_prep(VxArgs v) {
  __shared__ uint32_t wsum[33];
  __shared__ uint32_t carry_t;
  __shared__ unsigned long long carry_w;
  if (threadIdx.x == 0) {
    carry_t = 0;
    carry_w = 0;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint32_t b0 = 0; b0 < v.n_samples; b0 += blockDim.x) {
    const uint32_t s = b0 + threadIdx.x;
    uint32_t n = 0, tiles = 0;
    if (s < v.n_samples) {
      VxCloud& c = v.cl[s];
      const uint32_t* h = hdr(v, v.A, s);
      c.active = 0;
      c.status = (int32_t)h[0];
      if (h[0] == (uint32_t)kOk) {
        n = h[2 + v.role_data];
        const uint32_t present = h[1];
        // range_crop / voxel check_move (kernels.cu): every moved field holds
        // at least as many points as "data"
        int32_t st = kOk;
        for (int f = 0; f < v.n_bytes_fields; ++f)
          if (((v.mm & present) >> f) & 1u)
            if (h[2 + f] < n) st = kOutOfBounds;
        if (st != kOk) {
          c.status = st;
          c.fail_op = v.vx_first + 1;
          n = 0;
        } else {
          c.active = 1;
          tiles = (n + kTile - 1) / kTile;
        }
      }
      c.n = n;
      c.n_tiles = tiles;
      c.mn[0] = c.mn[1] = c.mn[2] = 0xffffffffu;
      c.mx[0] = c.mx[1] = c.mx[2] = 0u;
    }
    // exclusive scans of tiles and points over samples
    const uint32_t ti = warp_incl_scan(tiles), pi = warp_incl_scan(n);
    if (lane == 31) wsum[w] = ti;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      for (uint32_t k = 0; k < nw; ++k) {
        const uint32_t c = wsum[k];
        wsum[k] = acc;
        acc += c;
      }
    }
    __syncthreads();
    const uint32_t t0 = carry_t + wsum[w] + ti - tiles;
    __syncthreads();
    if (lane == 31) wsum[w] = pi;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      for (uint32_t k = 0; k < nw; ++k) {
        const uint32_t c = wsum[k];
        wsum[k] = acc;
        acc += c;
      }
    }
    __syncthreads();
    const uint64_t p0 = carry_w + wsum[w] + pi - n;
    if (s < v.n_samples) {
      v.cl[s].tile0 = t0;
      v.cl[s].word0 = p0;
      for (uint32_t k = 0; k < tiles; ++k) v.tile_cloud[t0 + k] = s;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry_t = t0 + tiles;
      carry_w = p0 + n;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *v.total_tiles = carry_t;
}

// ---------------------------------------------------------------- bounds
__global__ void __launch_bounds__(kThreads) k_vx_bounds(VxArgs v) {
  __shared__ uint32_t red[kWarps][8];
  const uint32_t total = *v.total_tiles;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t s = v.tile_cloud[t];
    VxCloud& c = v.cl[s];
    const float* d = reinterpret_cast<const float*>(slot(v, v.A, s) + v.off[v.role_data]);
    const uint32_t i0 = (t - c.tile0) * kTile;
    uint32_t mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[3] = {0, 0, 0};
    uint32_t kept = 0, nan = 0;
    float p[kItems][3];
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t i = i0 + r * kThreads + threadIdx.x;
#pragma unroll
      for (int a = 0; a < 3; ++a) p[r][a] = i < c.n ? d[3ull * i + a] : 0.0f;
    }
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t i = i0 + r * kThreads + threadIdx.x;
      if (i < c.n && in_box(v, p[r][0], p[r][1], p[r][2])) {
        ++kept;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (isnan(p[r][a])) nan = 1;
          else {
            mn[a] = min(mn[a], ord_f(p[r][a]));
            mx[a] = max(mx[a], ord_f(p[r][a]));
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kept += __shfl_xor_sync(0xffffffffu, kept, o);
      nan |= __shfl_xor_sync(0xffffffffu, nan, o);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
        mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
      }
    }
    if (lane == 0) {
      red[w][0] = kept;
      red[w][1] = nan;
      for (int a = 0; a < 3; ++a) {
        red[w][2 + a] = mn[a];
        red[w][5 + a] = mx[a];
      }
    }
    __syncthreads();
    if (threadIdx.x < 8) {
      const uint32_t k = threadIdx.x;
      uint32_t x = red[0][k];
      for (uint32_t q = 1; q < kWarps; ++q) {
        const uint32_t y = red[q][k];
        x = k == 0 ? x + y : k == 1 ? (x | y) : k < 5 ? min(x, y) : max(x, y);
      }
      if (k == 0) v.tile_kept[t] = x;
      else if (k == 1) { if (x) atomicOr(&c.nan, 1u); }
      else if (k < 5) { if (x != 0xffffffffu) atomicMin(&c.mn[k - 2], x); }
      else atomicMax(&c.mx[k - 5], x);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- plan
__global__ void __launch_bounds__(kThreads) k_vx_plan(VxArgs v) {
  __shared__ uint32_t sh[kWarps + 1];
  __shared__ uint32_t carry;
  const uint32_t s = blockIdx.x;
  VxCloud& c = v.cl[s];
  if (!c.active) return;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t j0 = 0; j0 < c.n_tiles; j0 += kThreads) {
    const uint32_t j = j0 + threadIdx.x;
    const uint32_t x = j < c.n_tiles ? v.tile_kept[c.tile0 + j] : 0;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(x, sh, &tot);
    if (j < c.n_tiles) v.tile_kofs[c.tile0 + j] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const uint32_t kept = carry;
  c.kept = kept;
  int32_t st = kOk;
  if (kept == 0) st = kEmptyCloud;  // run_chain: the voxel op sees zero points
  else if (c.nan) st = kOutOfBounds;
  uint32_t q0[3] = {0, 0, 0}, q1[3] = {0, 0, 0};
  if (st == kOk) {
    for (int a = 0; a < 3; ++a) {
      const float o = v.has_origin ? v.origin[a] : unord_f(c.mn[a]);
      c.o[a] = o;
      const float lo = qkey(unord_f(c.mn[a]), o, v.voxel), hi = qkey(unord_f(c.mx[a]), o, v.voxel);
      // keys are monotone in the coordinate: the extremes bound every key
      if (!(lo >= 0.0f && lo < 2097152.0f && hi >= 0.0f && hi < 2097152.0f)) st = kOutOfBounds;
      else {
        q0[a] = (uint32_t)lo;
        q1[a] = (uint32_t)hi;
      }
    }
  }
  c.status = st;
  c.fail_op = st == kOk ? 0 : v.vx_last + 1;
  if (st != kOk) {
    c.active = 0;
    return;
  }
  uint32_t kb = 0;
  for (int a = 0; a < 3; ++a) {
    const uint32_t span = q1[a] - q0[a];
    c.q0[a] = q0[a];
    c.bx[a] = span ? 32u - __clz(span) : 0u;
    kb += c.bx[a];
  }
  const uint32_t ib = c.n > 1 ? 32u - __clz(c.n - 1) : 0u;
  c.kb = kb;
  c.ib = ib;
  c.passes = (kb + 7) / 8;
  if (kb + ib > 64 || c.passes > kVxMaxPasses) {  // k_cloud's op_voxel handles it
    c.fallback = 1;
    c.active = 0;
  }
}

// ---------------------------------------------------------------- keys
__global__ void __launch_bounds__(kThreads) k_vx_keys(VxArgs v) {
  __shared__ uint32_t sh[kWarps + 1];
  __shared__ uint32_t hist[kVxMaxPasses][256];
  const uint32_t total = *v.total_tiles;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t s = v.tile_cloud[t];
    const VxCloud& c = v.cl[s];
    if (!c.active) continue;  // uniform
    for (uint32_t k = threadIdx.x; k < c.passes * 256; k += kThreads) (&hist[0][0])[k] = 0;
    const float* d = reinterpret_cast<const float*>(slot(v, v.A, s) + v.off[v.role_data]);
    const uint32_t i0 = (t - c.tile0) * kTile + threadIdx.x * kItems;  // thread-contiguous: order-preserving scan
    float p[kItems][3];
    uint32_t keep = 0;
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t i = i0 + r;
#pragma unroll
      for (int a = 0; a < 3; ++a) p[r][a] = i < c.n ? d[3ull * i + a] : 0.0f;
      if (i < c.n && in_box(v, p[r][0], p[r][1], p[r][2])) keep |= 1u << r;
    }
    uint32_t tot;
    uint32_t pos = block_excl_scan(__popc(keep), sh, &tot);
    uint64_t* out = v.w0 + c.word0 + v.tile_kofs[t];
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      if (!((keep >> r) & 1u)) continue;
      uint64_t key = 0;
      uint32_t sh_bits = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const uint32_t q = (uint32_t)qkey(p[r][a], c.o[a], v.voxel) - c.q0[a];
        key |= (uint64_t)q << sh_bits;
        sh_bits += c.bx[a];
      }
      const uint64_t word = (key << c.ib) | (uint64_t)(i0 + r);
      out[pos++] = word;
      for (uint32_t ps = 0; ps < c.passes; ++ps) atomicAdd(&hist[ps][(word >> (c.ib + 8 * ps)) & 255u], 1u);
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < c.passes * 256; k += kThreads) {
      const uint32_t x = (&hist[0][0])[k];
      if (x) atomicAdd(&v.cl[s].hist[k >> 8][k & 255u], x);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- sort
// Tile j of cloud c covers words [j*kTile, min((j+1)*kTile, kept)).
// pass = -1: any active cloud (segments / means after the last pass).
__device__ __forceinline__ bool sort_tile(const VxArgs& v, uint32_t t, int pass, uint32_t& s,
                                          uint32_t& j, uint32_t& n_w) {
  s = v.tile_cloud[t];
  const VxCloud& c = v.cl[s];
  if (!c.active || (pass >= 0 && (uint32_t)pass >= c.passes)) return false;
  j = t - c.tile0;
  const uint32_t w0 = j * kTile;
  if (w0 >= c.kept) return false;
  n_w = min(kTile, c.kept - w0);
  return true;
}

__global__ void __launch_bounds__(kThreads) k_vx_upsweep(VxArgs v, uint32_t pass) {
  __shared__ uint32_t h[256];
  const uint32_t total = *v.total_tiles;
  const uint64_t* src = (pass & 1u) ? v.w1 : v.w0;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    uint32_t s, j, nw;
    if (!sort_tile(v, t, (int)pass, s, j, nw)) continue;  // uniform
    const VxCloud& c = v.cl[s];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t* in = src + c.word0 + (uint64_t)j * kTile;
    const uint32_t shb = c.ib + 8 * pass;
    uint64_t x[kItems];
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t i = r * kThreads + threadIdx.x;
      x[r] = i < nw ? in[i] : 0;
    }
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r)
      if (r * kThreads + threadIdx.x < nw) atomicAdd(&h[(x[r] >> shb) & 255u], 1u);
    __syncthreads();
    v.cnt[(uint64_t)t * 256 + threadIdx.x] = h[threadIdx.x];
    __syncthreads();
  }
}

// grid (n_samples, 8): warp w of CTA y scans digit 32*y + w over the cloud's
// sort tiles: cnt[t][d] := base[d] + sum of cnt[t'][d] for t' < t.
__global__ void __launch_bounds__(1024) k_vx_colscan(VxArgs v, uint32_t pass) {
  const uint32_t s = blockIdx.x;
  const VxCloud& c = v.cl[s];
  if (!c.active || pass >= c.passes) return;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t d = blockIdx.y * 32 + w;
  // digit base: cloud-wide count of smaller digits
  uint32_t b = 0;
  for (uint32_t k = lane; k < d; k += 32) b += c.hist[pass][k];
#pragma unroll
  for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  const uint32_t tiles = (c.kept + kTile - 1) / kTile;
  uint32_t carry = b;
  for (uint32_t j0 = 0; j0 < tiles; j0 += 32) {
    const uint32_t j = j0 + lane;
    uint32_t* p = v.cnt + (uint64_t)(c.tile0 + j) * 256 + d;
    const uint32_t x = j < tiles ? *p : 0;
    const uint32_t inc = warp_incl_scan(x);
    if (j < tiles) *p = carry + inc - x;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// Stable scatter of one tile: warp q owns the tile's words [q*256, q*256+256)
// in 8 rounds of 32 (lane order = word order); per-warp digit counts (match
// ranks), then per (digit, warp) bases from the tile's scanned offsets.
__global__ void __launch_bounds__(kThreads) k_vx_downsweep(VxArgs v, uint32_t pass) {
  __shared__ uint32_t wc[kWarps][256];
  const uint32_t total = *v.total_tiles;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t* src = (pass & 1u) ? v.w1 : v.w0;
  uint64_t* dst = (pass & 1u) ? v.w0 : v.w1;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    uint32_t s, j, nw;
    if (!sort_tile(v, t, (int)pass, s, j, nw)) continue;  // uniform
    const VxCloud& c = v.cl[s];
    const uint64_t* in = src + c.word0 + (uint64_t)j * kTile;
    const uint32_t shb = c.ib + 8 * pass;
    uint32_t* row = wc[w];
    for (uint32_t k = lane; k < 256; k += 32) row[k] = 0;
    __syncwarp();
    uint64_t x[kItems];
    uint32_t dg[kItems];
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t i = w * 256 + r * 32 + lane;
      x[r] = i < nw ? in[i] : 0;
      dg[r] = i < nw ? (uint32_t)((x[r] >> shb) & 255u) : 256u;
    }
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t peers = __match_any_sync(0xffffffffu, dg[r]);
      if (dg[r] < 256u && (peers & lt) == 0) row[dg[r]] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // bases: tile offset of the digit + counts of the same digit in earlier warps
    {
      const uint32_t d = threadIdx.x;  // kThreads == 256 digits
      uint32_t acc = v.cnt[(uint64_t)t * 256 + d];
      for (uint32_t q = 0; q < kWarps; ++q) {
        const uint32_t cq = wc[q][d];
        wc[q][d] = acc;
        acc += cq;
      }
    }
    __syncthreads();
    uint64_t* out = dst + c.word0;
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t peers = __match_any_sync(0xffffffffu, dg[r]);
      if (dg[r] < 256u) {
        const uint32_t pos = row[dg[r]] + __popc(peers & lt);
        out[pos] = x[r];
      }
      __syncwarp();
      if (dg[r] < 256u && (peers & lt) == 0) row[dg[r]] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- segments
__device__ __forceinline__ const uint64_t* sorted(const VxArgs& v, const VxCloud& c) {
  return ((c.passes & 1u) ? v.w1 : v.w0) + c.word0;
}

__global__ void __launch_bounds__(kThreads) k_vx_segcount(VxArgs v) {
  __shared__ uint32_t sh[kWarps + 1];
  const uint32_t total = *v.total_tiles;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    uint32_t s, j, nw;
    if (!sort_tile(v, t, -1, s, j, nw)) {
      v.tile_kept[t] = 0;
      continue;
    }
    const VxCloud& c = v.cl[s];
    const uint64_t* W = sorted(v, c);
    const uint32_t base = j * kTile;
    uint32_t cnt = 0;
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t i = base + r * kThreads + threadIdx.x;
      if (i < base + nw && (i == 0 || (W[i] >> c.ib) != (W[i - 1] >> c.ib))) ++cnt;
    }
    uint32_t tot;
    block_excl_scan(cnt, sh, &tot);
    if (threadIdx.x == 0) v.tile_kept[t] = tot;  // reused: voxel starts per tile
  }
}

__global__ void __launch_bounds__(kThreads) k_vx_segscan(VxArgs v) {
  __shared__ uint32_t sh[kWarps + 1];
  __shared__ uint32_t carry;
  const uint32_t s = blockIdx.x;
  VxCloud& c = v.cl[s];
  if (!c.active) return;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t tiles = (c.kept + kTile - 1) / kTile;
  for (uint32_t j0 = 0; j0 < tiles; j0 += kThreads) {
    const uint32_t j = j0 + threadIdx.x;
    const uint32_t x = j < tiles ? v.tile_kept[c.tile0 + j] : 0;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(x, sh, &tot);
    if (j < tiles) v.tile_kofs[c.tile0 + j] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) c.V = carry;
}

// Payload of every moved field into sorted order: B[f][k] = A[f][index(k)]
// (one sorted position per thread per round: coalesced word reads and
// stores, independent random loads -- many in flight).
__global__ void __launch_bounds__(kThreads) k_vx_gather(VxArgs v) {
  const uint32_t total = *v.total_tiles;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    uint32_t s, j, nw;
    if (!sort_tile(v, t, -1, s, j, nw)) continue;  // uniform
    const VxCloud& c = v.cl[s];
    const uint64_t* W = sorted(v, c) + (uint64_t)j * kTile;
    const uint8_t* A = slot(v, v.A, s);
    uint8_t* B = v.B + (uint64_t)s * v.stride;
    const uint32_t* ha = hdr(v, v.A, s);
    const uint32_t moved = v.mm & ha[1];
    const uint64_t imask = c.ib ? ((1ull << c.ib) - 1) : 0ull;
    uint32_t idx[kItems];
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t i = r * kThreads + threadIdx.x;
      idx[r] = i < nw ? (uint32_t)(W[i] & imask) : 0u;
    }
    const uint64_t k0 = (uint64_t)j * kTile;
    for (int f = 0; f < v.n_bytes_fields; ++f) {
      if (!((moved >> f) & 1u)) continue;
      const uint32_t es = ha[10 + f];
      if (es == 12) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(A + v.off[f]);
        uint32_t* dst = reinterpret_cast<uint32_t*>(B + v.off[f]);
        uint32_t x[kItems][3];
#pragma unroll
        for (uint32_t r = 0; r < kItems; ++r)
          if (r * kThreads + threadIdx.x < nw)
#pragma unroll
            for (int q = 0; q < 3; ++q) x[r][q] = src[3ull * idx[r] + q];
#pragma unroll
        for (uint32_t r = 0; r < kItems; ++r) {
          const uint32_t i = r * kThreads + threadIdx.x;
          if (i < nw)
#pragma unroll
            for (int q = 0; q < 3; ++q) dst[3 * (k0 + i) + q] = x[r][q];
        }
      } else if (es == 4) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(A + v.off[f]);
        uint32_t* dst = reinterpret_cast<uint32_t*>(B + v.off[f]);
        uint32_t x[kItems];
#pragma unroll
        for (uint32_t r = 0; r < kItems; ++r)
          if (r * kThreads + threadIdx.x < nw) x[r] = src[idx[r]];
#pragma unroll
        for (uint32_t r = 0; r < kItems; ++r) {
          const uint32_t i = r * kThreads + threadIdx.x;
          if (i < nw) dst[k0 + i] = x[r];
        }
      } else {
        const uint8_t* src = A + v.off[f];
        uint8_t* dst = B + v.off[f];
        for (uint32_t r = 0; r < kItems; ++r) {
          const uint32_t i = r * kThreads + threadIdx.x;
          if (i < nw)
            for (uint32_t b = 0; b < es; ++b) dst[(k0 + i) * es + b] = src[(uint64_t)idx[r] * es + b];
        }
      }
    }
  }
}

// One thread per voxel start (thread-contiguous items, so the block scan
// numbers the tile's starts in order): count and sequential double sums over
// the voxel's contiguous sorted run in B (point order inside the voxel),
// means / first point written to A at the voxel index (A's payload is dead
// after k_vx_gather; the voxelized cloud lives in A from here on).
__global__ void __launch_bounds__(kThreads) k_vx_means(VxArgs v) {
  __shared__ uint32_t sh[kWarps + 1];
  const uint32_t total = *v.total_tiles;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    uint32_t s, j, nw;
    if (!sort_tile(v, t, -1, s, j, nw)) continue;  // uniform
    const VxCloud& c = v.cl[s];
    const uint64_t* W = sorted(v, c);
    const uint32_t base = j * kTile + threadIdx.x * kItems;
    const uint32_t end = j * kTile + nw;
    uint32_t starts = 0;
    uint64_t prev = base ? W[base - 1] >> c.ib : ~0ull;
#pragma unroll
    for (uint32_t r = 0; r < kItems; ++r) {
      const uint32_t i = base + r;
      if (i < end) {
        const uint64_t key = W[i] >> c.ib;
        if (i == 0 || key != prev) starts |= 1u << r;
        prev = key;
      }
    }
    uint32_t tot;
    uint32_t vid = v.tile_kofs[t] + block_excl_scan(__popc(starts), sh, &tot);
    uint8_t* A = v.A + (uint64_t)s * v.stride;
    const uint8_t* B = v.B + (uint64_t)s * v.stride;
    const uint32_t* ha = hdr(v, v.A, s);
    const uint32_t moved = v.mm & ha[1];
    while (starts) {
      const uint32_t r = __ffs(starts) - 1;
      starts &= starts - 1;
      const uint32_t k0 = base + r;
      const uint64_t key = W[k0] >> c.ib;
      uint32_t k1 = k0 + 1;
      while (k1 < c.kept && (W[k1] >> c.ib) == key) ++k1;
      const double cnt = (double)(k1 - k0);
      for (int f = 0; f < v.n_bytes_fields; ++f) {
        if (!((moved >> f) & 1u)) continue;
        const bool avg = f == v.role_data || f == v.role_normal || f == v.role_color || f == v.role_intensity;
        const uint32_t es = ha[10 + f];
        if (avg) {
          const uint32_t comps = es / 4;  // 3 or 1
          const float* src = reinterpret_cast<const float*>(B + v.off[f]);
          float* dst = reinterpret_cast<float*>(A + v.off[f]);
          if (comps == 3) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0;
            for (uint32_t k = k0; k < k1; ++k) {
              a0 = __dadd_rn(a0, (double)src[3ull * k]);
              a1 = __dadd_rn(a1, (double)src[3ull * k + 1]);
              a2 = __dadd_rn(a2, (double)src[3ull * k + 2]);
            }
            dst[3ull * vid] = __double2float_rn(__ddiv_rn(a0, cnt));
            dst[3ull * vid + 1] = __double2float_rn(__ddiv_rn(a1, cnt));
            dst[3ull * vid + 2] = __double2float_rn(__ddiv_rn(a2, cnt));
          } else {
            double a0 = 0.0;
            for (uint32_t k = k0; k < k1; ++k) a0 = __dadd_rn(a0, (double)src[k]);
            dst[vid] = __double2float_rn(__ddiv_rn(a0, cnt));
          }
        } else {  // gathered extra field: the voxel's first point (smallest index)
          const uint8_t* src = B + v.off[f] + (uint64_t)k0 * es;
          uint8_t* dst = A + v.off[f] + (uint64_t)vid * es;
          for (uint32_t b = 0; b < es; ++b) dst[b] = src[b];
        }
      }
      if (v.counts) reinterpret_cast<int32_t*>(A + v.off[kMaxBytesFields])[vid] = (int32_t)(k1 - k0);
      ++vid;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- finish
__global__ void k_vx_finish(VxArgs v) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= v.n_samples) return;
  const VxCloud& c = v.cl[s];
  uint32_t* h = reinterpret_cast<uint32_t*>(v.A + (uint64_t)s * v.stride);
  // decode launch failed (it wrote the status) or fallback (A keeps the
  // decoded cloud; k_cloud runs the voxel ops): header unchanged
  if (h[0] != (uint32_t)kOk || c.fallback) return;
  if (c.status != kOk) {
    h[0] = (uint32_t)c.status;
    v.sample_status[s] = c.status;
    v.sample_op[s] = c.fail_op;
    v.sample_where[s] = 0;
    return;
  }
  for (int f = 0; f < kMaxBytesFields; ++f)
    if (((v.mm & h[1]) >> f) & 1u) h[2 + f] = c.V;
  h[18] = v.counts ? 1u : 0u;
  h[19] = v.counts ? c.V : 0u;
}

}  // namespace

cudaError_t launch_voxel_wave(const VxArgs& v, uint32_t tiles_bound, int sms, cudaStream_t st) {
  if (!v.n_samples) return cudaSuccess;
  cudaMemsetAsync(v.cl, 0, sizeof(VxCloud) * v.n_samples, st);
  k_vx_prep<<<1, 1024, 0, st>>>(v);
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(tiles_bound, (uint32_t)sms * 8));
  k_vx_bounds<<<grid, kThreads, 0, st>>>(v);
  k_vx_plan<<<v.n_samples, kThreads, 0, st>>>(v);
  k_vx_keys<<<grid, kThreads, 0, st>>>(v);
  for (uint32_t p = 0; p < v.max_passes; ++p) {
    k_vx_upsweep<<<grid, kThreads, 0, st>>>(v, p);
    k_vx_colscan<<<dim3(v.n_samples, 8), 1024, 0, st>>>(v, p);
    k_vx_downsweep<<<grid, kThreads, 0, st>>>(v, p);
  }
  k_vx_segcount<<<grid, kThreads, 0, st>>>(v);
  k_vx_segscan<<<v.n_samples, kThreads, 0, st>>>(v);
  k_vx_gather<<<grid, kThreads, 0, st>>>(v);
  k_vx_means<<<grid, kThreads, 0, st>>>(v);
  k_vx_finish<<<(v.n_samples + 127) / 128, 128, 0, st>>>(v);
  return cudaGetLastError();
}

uint32_t voxel_wave_tile_points() { return kTile; }

}  // namespace pcp
