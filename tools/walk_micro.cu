// Latency floor of a single-thread pointer walk through a shared-memory
// table (the LZ4 skim walker's chain), with the per-step position store
// going nowhere / to shared / to global.  Diagnostics only.
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(uint32_t* g, long long* out, int steps) {
  __shared__ uint32_t tab[4096];
  __shared__ uint32_t rec[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = 3u | (6u << 16);
  __syncthreads();
  if (MODE < 3 && threadIdx.x) return;
  uint32_t lp = 0, n = 0;
  if (MODE >= 3 && threadIdx.x) {  // other lanes/warps parked at the block barrier (decoder shape)
    __syncthreads();
    return;
  }
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const uint32_t x = tab[lp & 4095];
    const uint32_t a = x & 0xFFFFu, b = x >> 16;
    if (MODE == 1) { rec[n & 4095] = lp; rec[(n + 1) & 4095] = lp + a; }
    if (MODE == 2 || MODE == 3) { g[n] = lp; g[n + 1] = lp + a; }
    n += b ? 2u : 1u;
    lp += b ? b : a;
  }
  long long t1 = clock64();
  out[0] = t1 - t0;
  out[1] = lp + n + rec[lp & 4095];
  if (MODE >= 3) __syncthreads();
}
int main() {
  uint32_t* g; long long* o; cudaMalloc(&g, 1 << 24); cudaMalloc(&o, 64);
  long long h[2];
  k<0><<<1, 128>>>(g, o, 20000); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost); printf("no store: %.1f cyc/step\n", h[0] / 20000.0);
  k<1><<<1, 128>>>(g, o, 20000); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost); printf("sts     : %.1f cyc/step\n", h[0] / 20000.0);
  k<2><<<1, 128>>>(g, o, 20000); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost); printf("stg     : %.1f cyc/step\n", h[0] / 20000.0);
  k<3><<<1, 256>>>(g, o, 20000); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost); printf("stg, lanes parked at bar: %.1f cyc/step\n", h[0] / 20000.0);
  return 0;
}
