// device_sort.cuh — CTA-wide stable LSD radix sort of 64-bit words
// (shared by the per-cloud interpreter and the multi-CTA voxel stage).
#pragma once

#include <cstdint>

#include "pcp_internal.h"

namespace pcp {

// Stable LSD radix sort of 64-bit words on bits [lo, hi), 8-bit digits
// (voxel keys packed above the point index, so the words carry their own
// payload), warp-partitioned: warp w owns the contiguous chunk
// [w*per, (w+1)*per).  Per pass: (a) every warp counts its chunk's digits,
// (b) one exclusive prefix over (digit, warp) gives each warp its bases,
// (c) every warp scatters its chunk in order (__match_any_sync ranks against
// its own counter row) — three block barriers per pass instead of two per
// tile; chunks are contiguous and ordered by warp, so the sort is stable.
// U words per lane are loaded ahead.  `scr`: kSortScratchBytes.  Returns 1
// if the result is in w1, 0 if in w0.
template <int U>
__device__ int radix_sort8(uint64_t* w0, uint64_t* w1, uint32_t n, uint32_t lo, uint32_t hi,
                           uint32_t* scr) {
  uint32_t* dsum = scr;             // [32] per-warp scan partials
  uint32_t* wcnt = scr + 8 * 256;   // [16][256]: counts, then bases
  const uint32_t t = threadIdx.x, nt = blockDim.x, lane = t & 31, w = t >> 5, nw = nt >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t np = (hi - lo + 7) / 8;
  const uint32_t per = ((n + nw - 1) / nw + 31) & ~31u;
  const uint32_t c0 = min(w * per, n), c1 = min(c0 + per, n);
  uint64_t* src = w0;
  uint64_t* dst = w1;
  for (uint32_t p = 0; p < np; ++p) {
    const uint32_t sh = lo + 8 * p;
    uint32_t* row = wcnt + w * 256;
    for (uint32_t k = lane; k < 256; k += 32) row[k] = 0;
    __syncwarp();
    // (a) digit counts of this warp's chunk
    for (uint32_t i0 = c0; i0 < c1; i0 += 32 * U) {
      uint64_t x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + 32 * u + lane;
        x[u] = i < c1 ? src[i] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool valid = i0 + 32 * u + lane < c1;
        const uint32_t d = valid ? (uint32_t)((x[u] >> sh) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (valid && (peers & lt) == 0) row[d] += __popc(peers);
        __syncwarp();
      }
    }
    __syncthreads();
    // (b) bases in (digit, warp) order
    uint32_t tot = 0;
    if (t < 256)
      for (uint32_t q = 0; q < nw; ++q) tot += wcnt[q * 256 + t];
    uint32_t x = tot;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((int)lane >= o) x += y;
    }
    if (t < 256 && lane == 31) dsum[w] = x;
    __syncthreads();
    if (t < 256) {
      uint32_t acc = x - tot;
      for (uint32_t k = 0; k < w; ++k) acc += dsum[k];
      for (uint32_t q = 0; q < nw; ++q) {
        const uint32_t c = wcnt[q * 256 + t];
        wcnt[q * 256 + t] = acc;
        acc += c;
      }
    }
    __syncthreads();
    // (c) scatter this warp's chunk in order
    for (uint32_t i0 = c0; i0 < c1; i0 += 32 * U) {
      uint64_t x2[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + 32 * u + lane;
        x2[u] = i < c1 ? src[i] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool valid = i0 + 32 * u + lane < c1;
        const uint32_t d = valid ? (uint32_t)((x2[u] >> sh) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & lt);
        const uint32_t pos = valid ? row[d] + rank : 0u;
        __syncwarp();
        if (valid) {
          dst[pos] = x2[u];
          if (rank == 0) row[d] += __popc(peers);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    uint64_t* tmp = src;
    src = dst;
    dst = tmp;
  }
  return (int)(np & 1u);
}


}  // namespace pcp
