// device_util.cuh — small sm_100a building blocks: CTA reductions/scans,
// unaligned word loads, TMA bulk staging (cp.async.bulk + mbarrier).
#pragma once

#include <cstdint>

namespace pcp {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Exactness certificate of a float sum (voxel means): with every value a
// multiple of 2^emin and n * max|x| < 2^(53 + emin), every partial sum of
// every order is exact in double, so a parallel sum equals the sequential
// one bit for bit.  ebits (biased exponent) bounds ilogb from above, also for
// denormals, so the test is conservative.
struct SumCert {
  int emin = 1 << 20;
  uint32_t ebits = 0;
  bool any = false, finite = true;
  __device__ __forceinline__ void add(float x) {
    const uint32_t b = __float_as_uint(x) & 0x7fffffffu;
    if (!b) return;
    const uint32_t e = b >> 23;
    if (e == 255u) {
      finite = false;
      return;
    }
    any = true;
    ebits = e > ebits ? e : ebits;
    const uint32_t m = b & 0x7fffffu;
    const int lb = e == 0 ? -149 + __ffs(m) - 1 : (int)e - 150 + __ffs(m | 0x800000u) - 1;
    emin = lb < emin ? lb : emin;
  }
  __device__ __forceinline__ void warp_merge() {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const int e2 = __shfl_xor_sync(0xffffffffu, emin, o);
      const uint32_t b2 = __shfl_xor_sync(0xffffffffu, ebits, o);
      emin = e2 < emin ? e2 : emin;
      ebits = b2 > ebits ? b2 : ebits;
    }
    any = __any_sync(0xffffffffu, any);
    finite = __all_sync(0xffffffffu, finite);
  }
  __device__ __forceinline__ bool exact(uint32_t n) const {
    const int nbits = 32 - __clz(n);
    return finite && (!any || (int)ebits - 127 + 1 + nbits <= 53 + emin);
  }
};

// 32-bit little-endian load from an arbitrarily aligned generic address.
// Reads the aligned word after it too (all buffers carry >= 16 B of slack).
__device__ __forceinline__ uint32_t ld_u32_unaligned(const uint8_t* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t sh = (a & 3u) * 8u;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const uint32_t lo = w[0];
  if (sh == 0) return lo;
  return __funnelshift_r(lo, w[1], sh);
}

// ---- mbarrier + bulk copy (TMA 1-D) ---------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(__cvta_generic_to_global(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

// ---- thread-block clusters (DSMEM) ------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// All threads of all CTAs of the cluster (release / acquire).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// Shared::cluster address of the same variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(smem_u32(p)), "r"(rank));
  return d;
}
// Remote (or local) shared store that completes `bytes` on the mbarrier at
// `rbar` (a shared::cluster address in the same CTA as `raddr`).
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint32_t a, uint32_t b, uint32_t c,
                                            uint32_t d, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::
          "r"(raddr),
      "r"(a), "r"(b), "r"(c), "r"(d), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void st_async_b32(uint32_t raddr, uint32_t a, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   raddr),
               "r"(a), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) { return __uint_as_float(lds_u32(a)); }

// ---- CTA reductions (red: >= 64 x 8 B of shared scratch) ------------------
template <typename T, typename Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T ident, void* red_) {
  T* red = reinterpret_cast<T*>(red_);
  const int t = threadIdx.x, nw = (blockDim.x + 31) >> 5;
  v = warp_reduce(v, op);
  __syncthreads();
  if ((t & 31) == 0) red[t >> 5] = v;
  __syncthreads();
  T r = (t & 31) < nw ? red[t & 31] : ident;
  r = warp_reduce(r, op);
  return r;  // every thread holds the result
}

struct OpAdd {
  template <typename T>
  __device__ T operator()(T a, T b) const { return a + b; }
};
struct OpDAdd {  // double add, explicit rounding (order-free only when exact)
  __device__ double operator()(double a, double b) const { return __dadd_rn(a, b); }
};
struct OpMin {
  template <typename T>
  __device__ T operator()(T a, T b) const { return b < a ? b : a; }
};
struct OpMax {
  template <typename T>
  __device__ T operator()(T a, T b) const { return a < b ? b : a; }
};
struct OpOr {
  __device__ uint32_t operator()(uint32_t a, uint32_t b) const { return a | b; }
};
struct OpFMax {  // NaN-ignoring max
  __device__ double operator()(double a, double b) const { return fmax(a, b); }
};

// Exclusive scan of v over the CTA; returns the prefix, *total = sum.
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* total, void* red_) {
  uint32_t* red = reinterpret_cast<uint32_t*>(red_);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = (blockDim.x + 31) >> 5;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[w] = x;
  __syncthreads();
  uint32_t base = 0, tot = 0;
  for (int i = 0; i < nw; ++i) {
    const uint32_t r = red[i];
    base += (i < w) ? r : 0;
    tot += r;
  }
  *total = tot;
  return base + x - v;
}

// argmax over (value, index): larger value wins, ties -> lower index, NaN
// never wins.  Index 0xFFFFFFFF = none.
struct ArgMax {
  float v;
  uint32_t i;
};
__device__ __forceinline__ bool argmax_better(float v, uint32_t i, float bv, uint32_t bi) {
  return v > bv || (v == bv && i < bi);
}
__device__ __forceinline__ ArgMax block_argmax(float v, uint32_t i, void* red_) {
  float* rv = reinterpret_cast<float*>(red_);
  uint32_t* ri = reinterpret_cast<uint32_t*>(rv + 32);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = (blockDim.x + 31) >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (argmax_better(ov, oi, v, i)) {
      v = ov;
      i = oi;
    }
  }
  __syncthreads();
  if (lane == 0) {
    rv[w] = v;
    ri[w] = i;
  }
  __syncthreads();
  float bv = lane < nw ? rv[lane] : -INFINITY;
  uint32_t bi = lane < nw ? ri[lane] : 0xFFFFFFFFu;
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (argmax_better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  return ArgMax{bv, bi};
}

}  // namespace dev
}  // namespace pcp
