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

#include "device_sort.cuh"
#include "device_util.cuh"
#include "voxel_wave.h"

namespace pcp {
namespace {

constexpr uint32_t kThreads = 256;
constexpr uint32_t kItems = 8;
constexpr uint32_t kTile = kThreads * kItems;  // points / words per tile
constexpr uint32_t kWarps = kThreads / 32;
constexpr uint32_t kBThreads = 512;  // bucket histogram / scatter
constexpr uint32_t kIThreads = 512;  // bucket-mode items

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

// Lowest-set-bit exponent of a finite nonzero float: x = odd * 2^e.
__device__ __forceinline__ int lowbit_exp(float x) {
  const uint32_t b = __float_as_uint(x) & 0x7fffffffu;
  const uint32_t e = b >> 23, m = b & 0x7fffffu;
  if (e == 0) return -149 + __ffs(m) - 1;
  return (int)e - 150 + __ffs(m | 0x800000u) - 1;
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
  __shared__ uint32_t carry_t, carry_b;
  __shared__ unsigned long long carry_w;
  if (threadIdx.x == 0) {
    carry_t = 0;
    carry_b = 0;
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
    __syncthreads();
    const uint32_t btiles = (n + kVxBTile - 1) / kVxBTile;
    const uint32_t bi = warp_incl_scan(btiles);
    if (lane == 31) wsum[w] = bi;
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
    const uint32_t bt0 = carry_b + wsum[w] + bi - btiles;
    if (s < v.n_samples) {
      v.cl[s].tile0 = t0;
      v.cl[s].word0 = p0;
      v.cl[s].btile0 = bt0;
      v.cl[s].n_btiles = btiles;
      for (uint32_t k = 0; k < tiles; ++k) v.tile_cloud[t0 + k] = s;
      for (uint32_t k = 0; k < btiles; ++k) v.btile_cloud[bt0 + k] = s;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry_t = t0 + tiles;
      carry_b = bt0 + btiles;
      carry_w = p0 + n;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *v.total_tiles = carry_t;
    *v.total_btiles = carry_b;
  }
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
  c.bb = kb < v.bucket_bits ? kb : v.bucket_bits;
  c.lowbits = kb - c.bb;
}

// ---------------------------------------------------------------- keys
__global__ void __launch_bounds__(kThreads) k_vx_keys(VxArgs v) {
  if (!*v.any_lsd) return;  // every cloud took the bucket mode
  __shared__ uint32_t sh[kWarps + 1];
  __shared__ uint32_t hist[kVxMaxPasses][256];
  const uint32_t total = *v.total_tiles;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t s = v.tile_cloud[t];
    const VxCloud& c = v.cl[s];
    if (!c.active || c.msd) continue;  // uniform (bucket-mode clouds skip the LSD path)
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
  if (!c.active || c.msd || (pass >= 0 && (uint32_t)pass >= c.passes)) return false;
  j = t - c.tile0;
  const uint32_t w0 = j * kTile;
  if (w0 >= c.kept) return false;
  n_w = min(kTile, c.kept - w0);
  return true;
}

__global__ void __launch_bounds__(kThreads) k_vx_upsweep(VxArgs v, uint32_t pass) {
  if (!*v.any_lsd) return;  // every cloud took the bucket mode
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
  if (!*v.any_lsd) return;  // every cloud took the bucket mode
  const uint32_t s = blockIdx.x;
  const VxCloud& c = v.cl[s];
  if (!c.active || c.msd || pass >= c.passes) return;
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
  if (!*v.any_lsd) return;  // every cloud took the bucket mode
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
  if (!*v.any_lsd) return;  // every cloud took the bucket mode
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
  if (!*v.any_lsd) return;  // every cloud took the bucket mode
  __shared__ uint32_t sh[kWarps + 1];
  __shared__ uint32_t carry;
  const uint32_t s = blockIdx.x;
  VxCloud& c = v.cl[s];
  if (!c.active || c.msd) return;
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
  if (!*v.any_lsd) return;  // every cloud took the bucket mode
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
  if (!*v.any_lsd) return;  // every cloud took the bucket mode
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

// ---------------------------------------------------------------- bucket mode
__device__ __forceinline__ uint64_t point_key(const VxArgs& v, const VxCloud& c, float x, float y, float z) {
  const float p[3] = {x, y, z};
  uint64_t key = 0;
  uint32_t sh_bits = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    key |= (uint64_t)((uint32_t)qkey(p[a], c.o[a], v.voxel) - c.q0[a]) << sh_bits;
    sh_bits += c.bx[a];
  }
  return key;
}

// Per scatter tile (kVxBTile points): bucket histogram of the kept points
// in shared memory, flushed into the cloud's bucket totals (one global atomic
// per non-empty bucket of the tile).
__global__ void __launch_bounds__(kBThreads) k_vx_bhist(VxArgs v) {
  __shared__ uint32_t h[kVxSmemBuckets];
  const uint32_t total = *v.total_btiles;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t s = v.btile_cloud[t];
    const VxCloud& c = v.cl[s];
    if (!c.active) continue;  // uniform
    const uint32_t nb = 1u << c.bb;
    const bool sm = nb <= kVxSmemBuckets;  // uniform
    uint32_t* tot = v.boff + (uint64_t)s * (v.bstride + 4);
    if (sm) {
      for (uint32_t k = threadIdx.x; k < nb; k += kBThreads) h[k] = 0;
      __syncthreads();
    }
    const float* d = reinterpret_cast<const float*>(slot(v, v.A, s) + v.off[v.role_data]);
    const uint32_t i0 = (t - c.btile0) * kVxBTile;
    const uint32_t i1 = min(c.n, i0 + kVxBTile);
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += kBThreads) {
      const float x = d[3ull * i], y = d[3ull * i + 1], z = d[3ull * i + 2];
      if (in_box(v, x, y, z)) {
        const uint32_t b = (uint32_t)(point_key(v, c, x, y, z) >> c.lowbits);
        if (sm) atomicAdd(&h[b], 1u);
        else atomicAdd(tot + b, 1u);  // many buckets: spread-address global reductions
      }
    }
    if (sm) {
      __syncthreads();
      for (uint32_t k = threadIdx.x; k < nb; k += kBThreads)
        if (h[k]) atomicAdd(tot + k, h[k]);
    }
    __syncthreads();
  }
}

// Per cloud: bucket offsets (exclusive scan of the totals), the write
// cursors (= offsets), the largest bucket, and the mode: bucket mode when the
// item sort word (key, point index, record position) fits 64 bits, else the
// global LSD sort (whose packed word may in turn not fit: then k_cloud's
// op_voxel runs the ops).
__global__ void __launch_bounds__(1024) k_vx_bbase(VxArgs v) {
  __shared__ uint32_t wsum[33];
  __shared__ uint32_t carry, mxs;
  const uint32_t s = blockIdx.x;
  VxCloud& c = v.cl[s];
  if (!c.active) return;
  const uint32_t nb = 1u << c.bb;
  uint32_t* bo = v.boff + (uint64_t)s * (v.bstride + 4);
  uint32_t* cur = v.bcur + (uint64_t)s * v.bstride;
  if (threadIdx.x == 0) carry = 0, mxs = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // chunks of 4 x 1024 buckets: 4 contiguous per thread (one 16-B load)
  for (uint32_t c0 = 0; c0 < nb; c0 += 4096) {
    const uint32_t b = c0 + 4 * threadIdx.x;
    uint4 x = make_uint4(0u, 0u, 0u, 0u);
    if (b + 3 < nb) x = *reinterpret_cast<const uint4*>(bo + b);
    else if (b < nb) {
      x.x = bo[b];
      if (b + 1 < nb) x.y = bo[b + 1];
      if (b + 2 < nb) x.z = bo[b + 2];
    }
    const uint32_t sum = x.x + x.y + x.z + x.w;
    uint32_t mx = max(max(x.x, x.y), max(x.z, x.w));
    const uint32_t inc = warp_incl_scan(sum);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 31) wsum[w] = inc;
    if (lane == 0) atomicMax(&mxs, mx);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = carry;
      for (uint32_t k = 0; k < 32; ++k) {
        const uint32_t cw = wsum[k];
        wsum[k] = acc;
        acc += cw;
      }
      wsum[32] = acc;
    }
    __syncthreads();
    uint32_t run = wsum[w] + inc - sum;
    const uint4 o = make_uint4(run, run + x.x, run + x.x + x.y, run + x.x + x.y + x.z);
    if (b + 3 < nb) {
      *reinterpret_cast<uint4*>(bo + b) = o;
      *reinterpret_cast<uint4*>(cur + b) = o;
    } else if (b < nb) {
      const uint32_t oo[4] = {o.x, o.y, o.z, o.w};
      for (uint32_t q = 0; b + q < nb; ++q) bo[b + q] = cur[b + q] = oo[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = wsum[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bo[nb] = carry;  // == kept
    c.max_bucket = mxs;
    const uint32_t pb = c.kept > 1 ? max(12u, 32u - __clz(c.kept - 1)) : 12u;  // item position bits, worst case
    const bool fits = v.msd_enabled && c.lowbits + c.bb + pb <= 64 && c.kb + c.ib <= 64;
    c.msd = fits ? 1u : 0u;
    c.n_items = fits ? c.kept / (kVxItemCap / 2) + 1 : 0;
    if (!fits) {
      atomicOr(v.any_lsd, 1u);
      if (c.kb + c.ib > 64 || c.passes > kVxMaxPasses) {  // k_cloud's op_voxel handles it
        c.fallback = 1;
        c.active = 0;
      }
    }
  }
  __syncthreads();
  // first bucket of every work item: item w starts at the first bucket whose
  // offset is >= w * half (nb when none is), i.e. bucket b starts the items
  // with bo[b-1] < w * half <= bo[b]
  if (!c.msd) return;
  constexpr uint32_t half = kVxItemCap / 2;
  uint32_t* ib = v.item_b + (uint64_t)s * v.max_items;
  for (uint32_t b = threadIdx.x; b <= nb; b += blockDim.x) {
    const uint32_t o = bo[b];
    const uint32_t wl = b ? bo[b - 1] / half + 1 : 0u;
    for (uint32_t w = wl; w <= o / half && w < c.n_items; ++w) ib[w] = b;
  }
}

// Scatter of a tile's kept points into their buckets: in-tile ranks from
// shared-memory atomics, one global atomic per non-empty bucket reserves the
// tile's run.  Order inside a bucket is not the point order; the item sort
// restores it (the word carries the point index).  Records: word = key << ib
// | index (w0), the payload of every moved field (B, same layout as A).
__global__ void __launch_bounds__(kBThreads) k_vx_bscatter(VxArgs v) {
  __shared__ uint32_t h[kVxSmemBuckets];
  constexpr uint32_t kPer = kVxBTile / kBThreads;
  const uint32_t total = *v.total_btiles;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t s = v.btile_cloud[t];
    const VxCloud& c = v.cl[s];
    if (!c.active || !c.msd) continue;  // uniform
    const uint32_t nb = 1u << c.bb;
    const bool sm = nb <= kVxSmemBuckets;  // uniform
    uint32_t* cur = v.bcur + (uint64_t)s * v.bstride;
    if (sm) {
      for (uint32_t k = threadIdx.x; k < nb; k += kBThreads) h[k] = 0;
      __syncthreads();
    }
    const float* d = reinterpret_cast<const float*>(slot(v, v.A, s) + v.off[v.role_data]);
    const uint32_t i0 = (t - c.btile0) * kVxBTile;
    uint64_t key[kPer];
    uint32_t rank[kPer];
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      const uint32_t i = i0 + q * kBThreads + threadIdx.x;
      rank[q] = ~0u;
      if (i < c.n) {
        const float x = d[3ull * i], y = d[3ull * i + 1], z = d[3ull * i + 2];
        if (in_box(v, x, y, z)) {
          key[q] = point_key(v, c, x, y, z);
          const uint32_t b = (uint32_t)(key[q] >> c.lowbits);
          rank[q] = sm ? atomicAdd(&h[b], 1u) : atomicAdd(cur + b, 1u);  // in-tile rank / final position
        }
      }
    }
    if (sm) {
      __syncthreads();
      for (uint32_t k = threadIdx.x; k < nb; k += kBThreads)
        if (h[k]) h[k] = atomicAdd(cur + k, h[k]);  // the tile's run start in the bucket
      __syncthreads();
    }
    const uint8_t* A = slot(v, v.A, s);
    uint8_t* B = v.B + (uint64_t)s * v.stride;
    const uint32_t* ha = hdr(v, v.A, s);
    const uint32_t moved = v.mm & ha[1];
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      if (rank[q] == ~0u) continue;
      const uint32_t i = i0 + q * kBThreads + threadIdx.x;
      const uint32_t pos = sm ? h[key[q] >> c.lowbits] + rank[q] : rank[q];
      v.w0[c.word0 + pos] = (key[q] << c.ib) | i;
      for (int f = 0; f < v.n_bytes_fields; ++f) {
        if (!((moved >> f) & 1u)) continue;
        const uint32_t es = ha[10 + f];
        if (es == 12) {
          const uint32_t* src = reinterpret_cast<const uint32_t*>(A + v.off[f]) + 3ull * i;
          uint32_t* dst = reinterpret_cast<uint32_t*>(B + v.off[f]) + 3ull * pos;
          dst[0] = src[0];
          dst[1] = src[1];
          dst[2] = src[2];
        } else if ((es & 3u) == 0) {
          const uint32_t* src = reinterpret_cast<const uint32_t*>(A + v.off[f]) + (uint64_t)i * (es >> 2);
          uint32_t* dst = reinterpret_cast<uint32_t*>(B + v.off[f]) + (uint64_t)pos * (es >> 2);
          for (uint32_t w = 0; w < (es >> 2); ++w) dst[w] = src[w];
        } else {
          for (uint32_t w = 0; w < es; ++w) B[v.off[f] + (uint64_t)pos * es + w] = A[v.off[f] + (uint64_t)i * es + w];
        }
      }
    }
    __syncthreads();
  }
}

// Work item w of a cloud: the buckets whose offset falls in
// [w * half, (w + 1) * half), at most kVxItemCap records (first buckets
// precomputed by k_vx_bbase).
__device__ __forceinline__ void item_range(const VxArgs& v, const VxCloud& c, uint32_t s, uint32_t w,
                                           uint32_t& b0, uint32_t& r0, uint32_t& r1) {
  const uint32_t nb = 1u << c.bb;
  const uint32_t* bo = v.boff + (uint64_t)s * (v.bstride + 4);
  const uint32_t* ib = v.item_b + (uint64_t)s * v.max_items;
  b0 = ib[w];
  const uint32_t b1 = w + 1 < c.n_items ? ib[w + 1] : nb;
  r0 = b0 < nb ? bo[b0] : c.kept;
  r1 = b1 < nb ? bo[b1] : c.kept;
}

using Cert = dev::SumCert;

// grid (max_items, n_samples), kIThreads threads.  An item's records (keys
// cached in registers) are sorted by key in shared memory -- a counting sort
// with warp-aggregated atomics when the item spans <= 4096 keys (dense
// voxels: order inside a key is arbitrary), else radix passes; items above
// kVxItemCap records sort in global memory (w2).  The payload of the moved
// fields and the point indices are staged in sorted order in shared memory
// (for the counting sort in the same pass, from coalesced record-order
// reads), so every voxel's run is contiguous.  Each voxel is then reduced --
// count, first point (smallest index) for gathered extra fields, and per
// float component the double sum, order-free under an exactness certificate
// (every value a multiple of 2^emin and n * max|x| < 2^(53 + emin): every
// partial sum of every order is exact), else replayed in point order (the
// App. C sequence).  Results to T[r0 + voxel], compacted into A afterwards.
__global__ void __launch_bounds__(kIThreads) k_vx_item(VxArgs v) {
  extern __shared__ __align__(16) uint8_t dyn[];
  uint64_t* sw0 = reinterpret_cast<uint64_t*>(dyn);
  uint64_t* sw1 = sw0 + kVxItemCap;
  uint32_t* scr = reinterpret_cast<uint32_t*>(sw1 + kVxItemCap);
  uint32_t* pay = scr + kSortScratchBytes / 4;  // [kVxItemCap][v.pay_words]
  constexpr uint32_t kIWarps = kIThreads / 32;
  constexpr uint32_t kPer = kVxItemCap / kIThreads;  // records per thread (small items)
  __shared__ uint32_t sh[kIWarps + 1];
  __shared__ unsigned long long red[32];
  const uint32_t s = blockIdx.y, w = blockIdx.x;
  const VxCloud& c = v.cl[s];
  if (!c.active || !c.msd || w >= c.n_items) return;
  uint32_t b0, r0, r1;
  item_range(v, c, s, w, b0, r0, r1);
  const uint32_t m = r1 - r0;
  uint32_t* iv = v.item_v + (uint64_t)s * v.max_items;
  if (m == 0) {
    if (threadIdx.x == 0) iv[w] = 0;
    return;
  }
  const uint32_t lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const uint64_t kbase = (uint64_t)b0 << c.lowbits;  // words = key << ib | point index
  const uint64_t* K = v.w0 + c.word0 + r0;
  const uint64_t imask = c.ib ? ((1ull << c.ib) - 1) : 0ull;
  const bool big = m > kVxItemCap;
  const uint32_t pb = big ? 32u - __clz(m - 1) : 12u;  // record position bits
  uint64_t* a0 = big ? v.w2 + 2 * c.word0 + r0 : sw0;
  uint64_t* a1 = big ? v.w2 + 2 * c.word0 + c.n + r0 : sw1;
  uint8_t* B = v.B + (uint64_t)s * v.stride;
  const uint32_t* ha = hdr(v, v.A, s);
  const uint32_t moved = v.mm & ha[1];
  // payload words of the moved 4-byte-multiple fields: field f's words at fo[f]
  const uint32_t PW = v.pay_words;
  uint32_t fo[kMaxBytesFields];
  {
    uint32_t o = 0;
    for (int f = 0; f < v.n_bytes_fields; ++f) {
      fo[f] = o;
      if ((moved >> f) & 1u) o += (ha[10 + f] + 3) / 4;
    }
  }
  const bool staged = !big && PW > 0;
  auto stage = [&](uint32_t j, uint32_t k) {  // record j's payload to sorted slot k
    for (int f = 0; f < v.n_bytes_fields; ++f) {
      if (!((moved >> f) & 1u)) continue;
      const uint32_t es = ha[10 + f];
      if (es & 3u) continue;  // odd-sized extra fields are read from B directly
      const uint32_t wpp = es >> 2;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(B + v.off[f]) + (uint64_t)(r0 + j) * wpp;
      uint32_t* dst = pay + k * PW + fo[f];
      if (wpp == 3) {
        const uint32_t x0 = src[0], x1 = src[1], x2 = src[2];
        dst[0] = x0, dst[1] = x1, dst[2] = x2;
      } else {
        for (uint32_t q = 0; q < wpp; ++q) dst[q] = src[q];
      }
    }
  };
  uint64_t kw[kPer];
  unsigned long long kmax = 0;
  if (!big) {
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      const uint32_t j = threadIdx.x + q * kIThreads;
      kw[q] = j < m ? K[j] : 0ull;
      if (j < m) kmax = max(kmax, (unsigned long long)((kw[q] >> c.ib) - kbase));
    }
  } else {
    for (uint32_t j = threadIdx.x; j < m; j += kIThreads)
      kmax = max(kmax, (unsigned long long)((K[j] >> c.ib) - kbase));
  }
  kmax = dev::block_reduce(kmax, dev::OpMax{}, 0ull, red);
  const uint32_t relbits = kmax ? 64u - __clzll(kmax) : 0u;
  const uint64_t* S;
  uint32_t* seg;   // voxel starts (<= m entries): first half of the free buffer
  uint32_t* sidx = nullptr;  // point index per sorted slot: its second half
  if (!big && relbits <= 12) {
    // counting sort; ranks from warp-aggregated atomics (dense voxels put
    // most of a warp's records on one key)
    uint32_t* hist = scr;  // <= 4096 counters
    const uint32_t range = 1u << relbits;
    for (uint32_t k = threadIdx.x; k < range; k += kIThreads) hist[k] = 0;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t rel[kPer], peers[kPer];
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      const uint32_t j = threadIdx.x + q * kIThreads;
      rel[q] = j < m ? (uint32_t)((kw[q] >> c.ib) - kbase) : 0xffffffffu;
      peers[q] = __match_any_sync(0xffffffffu, rel[q]);
      if (j < m && (peers[q] & lt) == 0) atomicAdd(&hist[rel[q]], (uint32_t)__popc(peers[q]));
    }
    __syncthreads();
    {
      const uint32_t per = (range + kIThreads - 1) / kIThreads;  // <= 8
      uint32_t x[8], sum = 0;
      for (uint32_t q = 0; q < per; ++q) {
        const uint32_t k = threadIdx.x * per + q;
        x[q] = k < range ? hist[k] : 0u;
        sum += x[q];
      }
      const uint32_t inc = warp_incl_scan(sum);
      if (lane == 31) sh[wp] = inc;
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t k = 0; k < kIWarps; ++k) {
          const uint32_t cw = sh[k];
          sh[k] = acc;
          acc += cw;
        }
      }
      __syncthreads();
      uint32_t run = sh[wp] + inc - sum;
      for (uint32_t q = 0; q < per; ++q) {
        const uint32_t k = threadIdx.x * per + q;
        if (k < range) hist[k] = run;
        run += x[q];
      }
    }
    __syncthreads();
    seg = reinterpret_cast<uint32_t*>(sw0);
    sidx = seg + kVxItemCap;
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      const uint32_t j = threadIdx.x + q * kIThreads;
      const uint32_t leader = __ffs(peers[q]) - 1;
      uint32_t base = 0;
      if (j < m && lane == leader) base = atomicAdd(&hist[rel[q]], (uint32_t)__popc(peers[q]));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (j < m) {
        const uint32_t k = base + __popc(peers[q] & lt);
        sw1[k] = ((uint64_t)rel[q] << pb) | j;
        sidx[k] = (uint32_t)(kw[q] & imask);
        if (staged) stage(j, k);
      }
    }
    S = sw1;
  } else {
    if (!big) {
#pragma unroll
      for (uint32_t q = 0; q < kPer; ++q) {
        const uint32_t j = threadIdx.x + q * kIThreads;
        if (j < m) a0[j] = (((kw[q] >> c.ib) - kbase) << pb) | j;
      }
    } else {
      for (uint32_t j = threadIdx.x; j < m; j += kIThreads) a0[j] = (((K[j] >> c.ib) - kbase) << pb) | j;
    }
    __syncthreads();
    const int r = radix_sort8<4>(a0, a1, m, pb, pb + relbits, scr);
    S = r ? a1 : a0;
    seg = reinterpret_cast<uint32_t*>(r ? a0 : a1);
    if (!big) {
      __syncthreads();
      sidx = seg + kVxItemCap;
      const uint64_t pm = (1ull << pb) - 1;
      for (uint32_t k = threadIdx.x; k < m; k += kIThreads) {
        const uint32_t j = (uint32_t)(S[k] & pm);
        sidx[k] = (uint32_t)(K[j] & imask);
        if (staged) stage(j, k);
      }
    }
  }
  const uint64_t pmask = (1ull << pb) - 1;
  __syncthreads();
  // voxel starts, numbered in order: thread-contiguous ranges, one block scan
  uint32_t V;
  {
    const uint32_t per = (m + kIThreads - 1) / kIThreads;
    const uint32_t ja = min(m, threadIdx.x * per), jb = min(m, ja + per);
    uint32_t cnt = 0;
    for (uint32_t j = ja; j < jb; ++j) cnt += (j == 0 || (S[j] >> pb) != (S[j - 1] >> pb)) ? 1u : 0u;
    const uint32_t inc = warp_incl_scan(cnt);
    if (lane == 31) sh[wp] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      for (uint32_t k = 0; k < kIWarps; ++k) {
        const uint32_t cw = sh[k];
        sh[k] = acc;
        acc += cw;
      }
      sh[kIWarps] = acc;
    }
    __syncthreads();
    uint32_t vid = sh[wp] + inc - cnt;
    V = sh[kIWarps];
    for (uint32_t j = ja; j < jb; ++j)
      if (j == 0 || (S[j] >> pb) != (S[j - 1] >> pb)) seg[vid++] = j;
  }
  __syncthreads();
  // component q of field f at sorted position k
  auto comp = [&](int f, uint32_t comps, uint32_t k, uint32_t q) -> float {
    if (staged) return __uint_as_float(pay[k * PW + fo[f] + q]);
    return reinterpret_cast<const float*>(B + v.off[f])[((uint64_t)r0 + (S[k] & pmask)) * comps + q];
  };
  auto pidx = [&](uint32_t k) -> uint64_t { return sidx ? (uint64_t)sidx[k] : K[S[k] & pmask] & imask; };
  // thread per small voxel, warp per large voxel; results to T[r0 + voxel]
  uint8_t* T = v.T + (uint64_t)s * v.stride;
  constexpr uint32_t kWarpVoxel = 64;
  auto emit = [&](uint32_t vx, uint32_t s0, uint32_t s1, bool warp_mode) {
    const uint32_t n = s1 - s0;
    const uint32_t k0 = s0 + (warp_mode ? lane : 0), dk = warp_mode ? 32 : 1;
    uint32_t first = s0;
    uint64_t first_i = ~0ull;
    for (uint32_t k = k0; k < s1; k += dk) {
      const uint64_t i = pidx(k);
      if (i < first_i) first_i = i, first = k;
    }
    if (warp_mode)
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t oi = __shfl_xor_sync(0xffffffffu, first_i, o);
        const uint32_t ok = __shfl_xor_sync(0xffffffffu, first, o);
        if (oi < first_i) first_i = oi, first = ok;
      }
    const bool writer = !warp_mode || lane == 0;
    for (int f = 0; f < v.n_bytes_fields; ++f) {
      if (!((moved >> f) & 1u)) continue;
      const bool avg = f == v.role_data || f == v.role_normal || f == v.role_color || f == v.role_intensity;
      const uint32_t es = ha[10 + f];
      if (avg) {
        const uint32_t comps = es / 4;
        float* dst = reinterpret_cast<float*>(T + v.off[f]) + (uint64_t)(r0 + vx) * comps;
        for (uint32_t q0 = 0; q0 < comps; q0 += 4) {  // up to 4 components per pass
          const uint32_t nq = min(4u, comps - q0);
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          Cert ct[4];
          for (uint32_t k = k0; k < s1; k += dk) {
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
              if (u < nq) {
                const float x = comp(f, comps, k, q0 + u);
                acc[u] = __dadd_rn(acc[u], (double)x);
                ct[u].add(x);
              }
            }
          }
#pragma unroll
          for (uint32_t u = 0; u < 4; ++u) {
            if (u >= nq) continue;
            if (warp_mode) {
#pragma unroll
              for (int o = 16; o; o >>= 1) acc[u] = __dadd_rn(acc[u], __shfl_xor_sync(0xffffffffu, acc[u], o));
              ct[u].warp_merge();
            }
            if (!writer) continue;
            if (!ct[u].exact(n)) {  // replay in point order
              acc[u] = 0.0;
              uint64_t last = 0;
              bool any = false;
              for (uint32_t t2 = 0; t2 < n; ++t2) {
                uint64_t best = ~0ull;
                uint32_t bk = s0;
                for (uint32_t k = s0; k < s1; ++k) {
                  const uint64_t i = pidx(k);
                  if ((!any || i > last) && i < best) best = i, bk = k;
                }
                acc[u] = __dadd_rn(acc[u], (double)comp(f, comps, bk, q0 + u));
                last = best;
                any = true;
              }
            }
            dst[q0 + u] = __double2float_rn(__ddiv_rn(acc[u], (double)n));
          }
        }
      } else if (writer) {  // gathered extra field: the voxel's first point
        uint8_t* dst = T + v.off[f] + (uint64_t)(r0 + vx) * es;
        if (staged && !(es & 3u)) {
          for (uint32_t q = 0; q < es / 4; ++q)
            reinterpret_cast<uint32_t*>(dst)[q] = pay[first * PW + fo[f] + q];
        } else {
          const uint8_t* src = B + v.off[f] + ((uint64_t)r0 + (S[first] & pmask)) * es;
          for (uint32_t q = 0; q < es; ++q) dst[q] = src[q];
        }
      }
    }
    if (v.counts && writer) reinterpret_cast<int32_t*>(T + v.off[kMaxBytesFields])[r0 + vx] = (int32_t)n;
  };
  for (uint32_t vx = threadIdx.x; vx < V; vx += kIThreads) {
    const uint32_t s0 = seg[vx], s1 = vx + 1 < V ? seg[vx + 1] : m;
    if (s1 - s0 <= kWarpVoxel) emit(vx, s0, s1, false);
  }
  for (uint32_t vx = wp; vx < V; vx += kIWarps) {
    const uint32_t s0 = seg[vx], s1 = vx + 1 < V ? seg[vx + 1] : m;
    if (s1 - s0 > kWarpVoxel) emit(vx, s0, s1, true);
  }
  if (threadIdx.x == 0) iv[w] = V;
}

__global__ void __launch_bounds__(kThreads) k_vx_iscan(VxArgs v) {
  __shared__ uint32_t sh[kWarps + 1];
  __shared__ uint32_t carry;
  const uint32_t s = blockIdx.x;
  VxCloud& c = v.cl[s];
  if (!c.active || !c.msd) return;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  uint32_t* iv = v.item_v + (uint64_t)s * v.max_items;
  for (uint32_t j0 = 0; j0 < c.n_items; j0 += kThreads) {
    const uint32_t j = j0 + threadIdx.x;
    const uint32_t x = j < c.n_items ? iv[j] : 0;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(x, sh, &tot);
    if (j < c.n_items) iv[j] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) c.V = carry;
}

// grid (max_items, n_samples): voxel results of item w from T[r0 ..] to A at
// the item's voxel offset.
__global__ void __launch_bounds__(kThreads) k_vx_compact(VxArgs v) {
  const uint32_t s = blockIdx.y, w = blockIdx.x;
  const VxCloud& c = v.cl[s];
  if (!c.active || !c.msd || w >= c.n_items) return;
  uint32_t b0, r0, r1;
  item_range(v, c, s, w, b0, r0, r1);
  const uint32_t* iv = v.item_v + (uint64_t)s * v.max_items;
  const uint32_t vo = iv[w], vn = (w + 1 < c.n_items ? iv[w + 1] : c.V) - vo;
  if (!vn) return;
  const uint8_t* T = v.T + (uint64_t)s * v.stride;
  uint8_t* A = v.A + (uint64_t)s * v.stride;
  const uint32_t* ha = hdr(v, v.A, s);
  const uint32_t moved = v.mm & ha[1];
  for (int f = 0; f < v.n_bytes_fields; ++f) {
    if (!((moved >> f) & 1u)) continue;
    const uint32_t es = ha[10 + f];
    if ((es & 3u) == 0) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(T + v.off[f]) + (uint64_t)r0 * (es >> 2);
      uint32_t* dst = reinterpret_cast<uint32_t*>(A + v.off[f]) + (uint64_t)vo * (es >> 2);
      for (uint32_t k = threadIdx.x; k < vn * (es >> 2); k += kThreads) dst[k] = src[k];
    } else {
      for (uint32_t k = threadIdx.x; k < vn * es; k += kThreads)
        A[v.off[f] + (uint64_t)vo * es + k] = T[v.off[f] + (uint64_t)r0 * es + k];
    }
  }
  if (v.counts) {
    const int32_t* src = reinterpret_cast<const int32_t*>(T + v.off[kMaxBytesFields]) + r0;
    int32_t* dst = reinterpret_cast<int32_t*>(A + v.off[kMaxBytesFields]) + vo;
    for (uint32_t k = threadIdx.x; k < vn; k += kThreads) dst[k] = src[k];
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

size_t voxel_wave_item_smem(uint32_t pay_words) {
  return 2 * 8 * kVxItemCap + kSortScratchBytes + 4ull * kVxItemCap * pay_words;
}

cudaError_t launch_voxel_wave(const VxArgs& v, uint32_t tiles_bound, uint32_t btiles_bound, int sms,
                              cudaStream_t st) {
  if (!v.n_samples) return cudaSuccess;
  static const bool attrs = [] {
    cudaFuncSetAttribute(k_vx_item, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)voxel_wave_item_smem(kVxMaxPayWords));
    return true;
  }();
  (void)attrs;
  cudaMemsetAsync(v.cl, 0, sizeof(VxCloud) * v.n_samples, st);
  cudaMemsetAsync(v.boff, 0, 4ull * (v.bstride + 4) * v.n_samples, st);
  cudaMemsetAsync(v.any_lsd, 0, 4, st);
  k_vx_prep<<<1, 1024, 0, st>>>(v);
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(tiles_bound, (uint32_t)sms * 8));
  const uint32_t bgrid = std::max<uint32_t>(1, std::min<uint32_t>(btiles_bound, (uint32_t)sms * 4));
  k_vx_bounds<<<grid, kThreads, 0, st>>>(v);
  k_vx_plan<<<v.n_samples, kThreads, 0, st>>>(v);
  // bucket mode (decided per cloud by k_vx_bbase)
  k_vx_bhist<<<bgrid, kBThreads, 0, st>>>(v);
  k_vx_bbase<<<v.n_samples, 1024, 0, st>>>(v);
  k_vx_bscatter<<<bgrid, kBThreads, 0, st>>>(v);
  k_vx_item<<<dim3(v.max_items, v.n_samples), kIThreads, voxel_wave_item_smem(v.pay_words), st>>>(v);
  k_vx_iscan<<<v.n_samples, kThreads, 0, st>>>(v);
  k_vx_compact<<<dim3(v.max_items, v.n_samples), kThreads, 0, st>>>(v);
  // global LSD mode (the other clouds)
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
