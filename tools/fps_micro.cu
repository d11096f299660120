// FPS iteration anatomy: the register-resident loop of kernels.cu fps_reg
// with clock64 checkpoints (warp 0 lane 0 and the last warp) per stage.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fps_micro tools/fps_micro.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <random>

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
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

template <int P, int MODE>
__global__ void __launch_bounds__(512, 1) k(const float* dg, uint32_t N, uint32_t M, int32_t* idx,
                                             long long* tm, float nz) {
  extern __shared__ float d[];
  __shared__ uint64_t slot[64];
  if (threadIdx.x < 64) slot[threadIdx.x] = 0;
  for (uint32_t i = threadIdx.x; i < 3 * N; i += blockDim.x) d[i] = dg[3 * (size_t)N * blockIdx.x + i];
  __syncthreads();
  const uint32_t t = threadIdx.x, nt = blockDim.x, lane = t & 31, w = t >> 5, nw = nt >> 5;
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
  long long acc[6] = {0, 0, 0, 0, 0, 0};
  for (uint32_t it = 0; it < M; ++it) {
    long long c0 = clock64();
    if (t == 0) idx[blockIdx.x * M + it] = (int32_t)sel;
    const float sx = d[3 * sel], sy = d[3 * sel + 1], sz = d[3 * sel + 2];
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
    long long c1 = clock64();
    if (MODE == 3) {
      long long c2 = clock64();
      const uint32_t vb = bv >= 0.f ? __float_as_uint(bv) : 0u;
      const uint32_t wmax = __reduce_max_sync(0xffffffffu, vb);
      const uint32_t par = it & 1u;
      uint32_t* vslot = reinterpret_cast<uint32_t*>(slot);  // [2][16] values, [2][16] indices at +32
      if (lane == 0) vslot[par * 16 + w] = wmax;
      long long c3 = clock64();
      __syncthreads();
      long long c4 = clock64();
      const uint32_t gv = lane < nw ? vslot[par * 16 + lane] : 0u;
      const uint32_t gmax = __reduce_max_sync(0xffffffffu, gv);
      if (wmax == gmax) {  // warp-uniform: only warps holding the maximum search
        uint32_t bk = 31;
        if (vb == gmax && bv >= 0.f) {
#pragma unroll
          for (int k = 0; k < P; ++k) bk = min(bk, mind[k] == bv ? (uint32_t)k : 31u);
        }
        const uint32_t bi = bk < 31 ? t + bk * nt : 0xFFFFFFFFu;
        const uint32_t wi = __reduce_min_sync(0xffffffffu, bi);
        if (lane == 0) vslot[64 + par * 16 + w] = wi;
      }
      __syncthreads();
      const uint32_t ii = (lane < nw && gv == gmax) ? vslot[64 + par * 16 + lane] : 0xFFFFFFFFu;
      sel = __reduce_min_sync(0xffffffffu, ii);
      if (sel == 0xFFFFFFFFu) sel = 0;
      long long c5 = clock64();
      acc[0] += c1 - c0;
      acc[1] += c2 - c1;
      acc[2] += c3 - c2;
      acc[3] += c4 - c3;
      acc[4] += c5 - c4;
      continue;
    }
    if (MODE == 2) {
      // pair-level search: lowest pair whose max equals bv, then within it
      uint32_t bj = P / 2;
#pragma unroll
      for (int j = P / 2 - 1; j >= 0; --j)
        bj = fmaxf(mind[2 * j], mind[2 * j + 1]) == bv ? (uint32_t)j : bj;
      float m0 = 0.f;
#pragma unroll
      for (int j = 0; j < P / 2; ++j) m0 = (uint32_t)j == bj ? mind[2 * j] : m0;
      const uint32_t bk2 = 2 * bj + (m0 == bv ? 0u : 1u);
      long long c2 = clock64();
      const uint32_t vb = bv >= 0.f ? __float_as_uint(bv) : 0u;
      const uint32_t wmax = __reduce_max_sync(0xffffffffu, vb);
      unsigned long long* best = reinterpret_cast<unsigned long long*>(slot);  // [3]
      if (vb == wmax && bv >= 0.f)
        atomicMax(best + (it % 3), ((unsigned long long)vb << 32) | (0xFFFFFFFFu - (t + bk2 * nt)));
      long long c3 = clock64();
      __syncthreads();
      long long c4 = clock64();
      const unsigned long long g = best[it % 3];
      if (t == 0) best[(it + 2) % 3] = 0ull;
      sel = g ? 0xFFFFFFFFu - (uint32_t)g : 0u;
      long long c5 = clock64();
      acc[0] += c1 - c0;
      acc[1] += c2 - c1;
      acc[2] += c3 - c2;
      acc[3] += c4 - c3;
      acc[4] += c5 - c4;
      continue;
    }
    uint32_t bk = P;
    if (MODE != 1) {
#pragma unroll
      for (int k = P - 1; k >= 0; --k) bk = mind[k] == bv ? (uint32_t)k : bk;
    } else {
      bk = 0;
    }
    const uint32_t vb = bv >= 0.f ? __float_as_uint(bv) : 0u;
    const uint32_t bi = bv >= 0.f ? t + bk * nt : 0xFFFFFFFFu;
    long long c2 = clock64();
    const uint32_t wmax = __reduce_max_sync(0xffffffffu, vb);
    const uint32_t wi = __reduce_min_sync(0xffffffffu, vb == wmax ? bi : 0xFFFFFFFFu);
    const uint32_t par = it & 1u;
    if (lane == 0) slot[par * 16 + w] = ((uint64_t)wmax << 32) | wi;
    long long c3 = clock64();
    __syncthreads();
    long long c4 = clock64();
    const uint64_t g = lane < nw ? slot[par * 16 + lane] : 0ull;
    const uint32_t gv = (uint32_t)(g >> 32);
    const uint32_t gmax = __reduce_max_sync(0xffffffffu, gv);
    sel = __reduce_min_sync(0xffffffffu, (lane < nw && gv == gmax) ? (uint32_t)g : 0xFFFFFFFFu);
    if (sel == 0xFFFFFFFFu) sel = 0;
    long long c5 = clock64();
    acc[0] += c1 - c0;
    acc[1] += c2 - c1;
    acc[2] += c3 - c2;
    acc[3] += c4 - c3;
    acc[4] += c5 - c4;
  }
  if (blockIdx.x == 0 && (t == 0 || t == nt - 32)) {
    for (int q = 0; q < 5; ++q) tm[(t ? 8 : 0) + q] = acc[q];
  }
}

int main() {
  const uint32_t N = 10000, M = 4000, clouds = 148;
  std::vector<float> h(3 * (size_t)N * clouds);
  std::mt19937 g(1);
  std::uniform_real_distribution<float> u(-1, 1);
  for (auto& x : h) x = u(g);
  float* d;
  int32_t* idx;
  long long* tm;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&idx, (size_t)clouds * M * 4);
  cudaMalloc(&tm, 16 * 8);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * N);
    for (int r = 0; r < 2; ++r) {
      cudaMemset(tm, 0, 128);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      kern<<<clouds, 512, 12 * N>>>(d, N, M, idx, tm, -0.0f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      long long t[16];
      cudaMemcpy(t, tm, 128, cudaMemcpyDeviceToHost);
      if (r)
        printf("%-10s %.3f ms  %.0f cyc/it | w0: loop %lld search %lld redux+sts %lld bar %lld redux2 %lld | wlast: loop %lld search %lld redux+sts %lld bar %lld redux2 %lld  (%s)\n",
               name, ms, ms * 1965e3 / M, t[0] / M, t[1] / M, t[2] / M, t[3] / M, t[4] / M, t[8] / M,
               t[9] / M, t[10] / M, t[11] / M, t[12] / M, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(k<20, 0>, "full");
  run(k<20, 1>, "nosearch");
  run(k<20, 2>, "pair+atom");
  run(k<20, 3>, "2bar");
  // check: MODE 0 and MODE 2 indices agree
  {
    std::vector<int32_t> a((size_t)clouds * M), b((size_t)clouds * M);
    k<20, 0><<<clouds, 512, 12 * N>>>(d, N, M, idx, tm, -0.0f);
    cudaMemcpy(a.data(), idx, a.size() * 4, cudaMemcpyDeviceToHost);
    k<20, 3><<<clouds, 512, 12 * N>>>(d, N, M, idx, tm, -0.0f);
    cudaMemcpy(b.data(), idx, b.size() * 4, cudaMemcpyDeviceToHost);
    printf("indices equal: %d\n", (int)(a == b));
  }
  return 0;
}
