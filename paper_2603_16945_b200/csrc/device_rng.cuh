// device_rng.cuh — bit-exact device restatement of the reference's RNG stack:
// std::mt19937_64 seeded with mix_seed (transforms.cpp:82-96,114) feeding
// libstdc++-13 generate_canonical<float,24> (random.tcc:3349-3381),
// uniform_real_distribution<float> (random.h:1909), normal_distribution<float>
// (polar method, random.tcc:1811-1843) and uniform_int_distribution<size_t>
// (Lemire _S_nd, uniform_int_dist.h:257-281).
//
// B200 shape: the 312-word state lives in shared memory; one thread runs the
// serial seeding recurrence, the whole CTA runs the twist (two dependency
// phases of 156 independent words) and tempers 312 outputs in parallel.  All
// float arithmetic on decision paths uses explicit _rn intrinsics: the
// reference is built without FMA contraction.
#pragma once

#include <cstdint>

namespace pcp {
namespace rng {

constexpr int kN = 312;
constexpr int kM = 156;
constexpr uint64_t kMatA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLower = 0x000000007FFFFFFFull;

__host__ __device__ inline uint64_t mix1(uint64_t h, uint64_t v) {
  h += 0x9e3779b97f4a7c15ull + v;
  h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
  h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
  return h ^ (h >> 31);
}

// mix_seed, transforms.cpp:82-96.
__host__ __device__ inline uint64_t mix_seed(uint64_t base, uint64_t epoch,
                                             uint64_t index, uint64_t op) {
  uint64_t h = mix1(base, 0x706370ull);
  h = mix1(h, epoch);
  h = mix1(h, index);
  return mix1(h, op);
}

__device__ __forceinline__ uint64_t seed_step(uint64_t prev, uint32_t i) {
  return 6364136223846793005ull * (prev ^ (prev >> 62)) + i;
}

__device__ __forceinline__ uint64_t temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

__device__ __forceinline__ uint64_t twist_word(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t y = (a & kUpper) | (b & kLower);
  return c ^ (y >> 1) ^ ((y & 1) ? kMatA : 0ull);
}

// Serial seeding into st[0..311] (one thread).
__device__ inline void seed_state(uint64_t* st, uint64_t seed) {
  uint64_t x = seed;
  st[0] = x;
  for (uint32_t i = 1; i < kN; ++i) {
    x = seed_step(x, i);
    st[i] = x;
  }
}

// CTA-cooperative twist (all threads of the block must call it).  Phase A
// words 0..155 read only old state; phase B words 156..311 read the new
// words 0..155 (and word 311 reads the new word 0).
__device__ inline void twist_block(uint64_t* st) {
  const int t = threadIdx.x;
  const int nt = blockDim.x;
  uint64_t v[2];
  int cnt = 0;
  for (int i = t; i < kM; i += nt) v[cnt++ & 1] = twist_word(st[i], st[i + 1], st[i + kM]);
  __syncthreads();
  cnt = 0;
  for (int i = t; i < kM; i += nt) st[i] = v[cnt++ & 1];
  __syncthreads();
  cnt = 0;
  for (int i = kM + t; i < kN; i += nt)
    v[cnt++ & 1] = twist_word(st[i], st[(i + 1) % kN], st[i - kM]);
  __syncthreads();
  cnt = 0;
  for (int i = kM + t; i < kN; i += nt) st[i] = v[cnt++ & 1];
  __syncthreads();
}

// The first k (<= 8) outputs of a freshly seeded engine, on ONE thread,
// without materialising the whole state: output i needs new word i, i.e.
// old words i, i+1 and i+156 (i < 156).  `w` = >= 166 words of scratch
// (shared memory: the engine state buffer).
__device__ inline void first_outputs(uint64_t seed, int k, uint64_t* out, uint64_t* w) {
  uint64_t x = seed;
  w[0] = x;
  const int need = kM + k + 1;
  for (int i = 1; i < need; ++i) {
    x = seed_step(x, (uint32_t)i);
    w[i] = x;
  }
  for (int i = 0; i < k; ++i) out[i] = temper(twist_word(w[i], w[i + 1], w[i + kM]));
}

// generate_canonical<float,24>: (float)u * 2^-64, clamp to nextafter(1,0).
__device__ __forceinline__ float canonical(uint64_t u) {
  float r = __fmul_rn(__ull2float_rn(u), 5.42101086242752217e-20f);  // 2^-64 exact
  return r >= 1.0f ? 0x1.fffffep-1f : r;
}

// uniform_real_distribution<float>(a,b): canon * (b - a) + a, no FMA.
__device__ __forceinline__ float uniform_real(uint64_t u, float a, float b) {
  return __fadd_rn(__fmul_rn(canonical(u), __fsub_rn(b, a)), a);
}

// One polar attempt: x, y = 2*canon - 1 (float result of a double subtract,
// which rounds identically to a float subtract of exact operands).
__device__ __forceinline__ bool polar_attempt(uint64_t u0, uint64_t u1, float& x, float& y,
                                              float& r2) {
  x = __double2float_rn(__dadd_rn((double)__fmul_rn(2.0f, canonical(u0)), -1.0));
  y = __double2float_rn(__dadd_rn((double)__fmul_rn(2.0f, canonical(u1)), -1.0));
  r2 = __fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y));
  return !(r2 > 1.0f || r2 == 0.0f);
}

// mult = sqrt(-2 * log(r2) / r2).  logf differs from glibc's by ulps: the
// values (not the draw stream) are tolerance-checked.
__device__ __forceinline__ float polar_mult(float r2) {
  return __fsqrt_rn(__fdiv_rn(__fmul_rn(-2.0f, logf(r2)), r2));
}

// Lemire: returns false when the rare rejection branch is needed
// (low < range), in which case the caller takes the serial path.
__device__ __forceinline__ bool lemire_fast(uint64_t u, uint64_t range, uint64_t& r) {
  const uint64_t lo = u * range;
  r = __umul64hi(u, range);
  return lo >= range;
}

// Serial engine (one thread, state in caller memory) for rare paths.
struct Serial {
  uint64_t* st;
  int idx;
  __device__ void seed(uint64_t s) {
    seed_state(st, s);
    idx = kN;
  }
  __device__ void twist() {
    for (int i = 0; i < kN; ++i) st[i] = twist_word(st[i], st[(i + 1) % kN], st[(i + kM) % kN]);
    idx = 0;
  }
  __device__ uint64_t next() {
    if (idx >= kN) twist();
    return temper(st[idx++]);
  }
  // uniform_int_distribution<size_t>(a, b)
  __device__ uint64_t uniform_int(uint64_t a, uint64_t b) {
    const uint64_t range = b - a + 1;
    uint64_t u = next();
    uint64_t lo = u * range;
    if (lo < range) {
      const uint64_t thr = (0ull - range) % range;
      while (lo < thr) {
        u = next();
        lo = u * range;
      }
    }
    return __umul64hi(u, range) + a;
  }
};

}  // namespace rng
}  // namespace pcp
