// Calibration: per-match cost of the warp-serial match resolver pattern.
#include <cstdio>
#include <cstdint>
__global__ void k(const uint32_t* mo_a, const uint32_t* ml_a, const uint16_t* off_a, uint32_t M,
                  long long* cyc, uint8_t* out, int variant) {
  __shared__ __align__(16) uint8_t ring[16384];
  const uint32_t t = threadIdx.x;
  for (int i = t; i < 16384; i += 32) ring[i] = (uint8_t)i;
  __syncwarp();
  long long t0 = clock64();
  for (uint32_t base = 0; base < M; base += 32) {
    const uint32_t q = base + t;
    uint32_t r_mo = 0, r_ml = 0, r_off = 1;
    if (q < M) { r_mo = mo_a[q]; r_ml = ml_a[q]; r_off = off_a[q]; }
    const uint32_t cnt = min(32u, M - base);
    if (variant == 2 && cnt == 32) {
      uint32_t A[32], MO[32], ML[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t mo = __shfl_sync(0xffffffffu, r_mo, j);
        const uint32_t ml = __shfl_sync(0xffffffffu, r_ml, j);
        const uint32_t off = __shfl_sync(0xffffffffu, r_off, j);
        uint32_t r = t - off * __float2uint_rz(__fdividef((float)t + 0.5f, (float)off));
        r = off >= ml ? t : r;
        A[j] = (mo - off + r) & 16383;
        MO[j] = (mo + t) & 16383;
        ML[j] = ml;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint8_t v = ring[A[j]];
        if (t < ML[j]) ring[MO[j]] = v;
        __syncwarp();
      }
      continue;
    }
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint32_t mo = __shfl_sync(0xffffffffu, r_mo, j);
      const uint32_t ml = __shfl_sync(0xffffffffu, r_ml, j);
      const uint32_t off = __shfl_sync(0xffffffffu, r_off, j);
      const uint32_t a = mo - off;
      uint32_t r;
      if (variant == 0) {
        r = t - off * __float2uint_rz(__fdividef((float)t + 0.5f, (float)off));
        r = off >= ml ? t : r;
      } else {
        r = t < off ? t : t % off;
      }
      const uint8_t v = ring[(a + r) & 16383];
      if (t < ml) ring[(mo + t) & 16383] = v;
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (t == 0) { cyc[0] = t1 - t0; out[0] = ring[5]; }
}
int main() {
  const uint32_t M = 100000;
  uint32_t *mo, *ml; uint16_t* off;
  uint32_t* hmo = new uint32_t[M]; uint32_t* hml = new uint32_t[M]; uint16_t* hoff = new uint16_t[M];
  uint32_t pos = 100;
  for (uint32_t i = 0; i < M; ++i) { pos += 16; hmo[i] = pos; hml[i] = 4 + (i * 7) % 6; hoff[i] = 1 + (i * 13) % 60; pos += hml[i]; }
  cudaMalloc(&mo, M * 4); cudaMalloc(&ml, M * 4); cudaMalloc(&off, M * 2);
  cudaMemcpy(mo, hmo, M * 4, cudaMemcpyHostToDevice); cudaMemcpy(ml, hml, M * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(off, hoff, M * 2, cudaMemcpyHostToDevice);
  long long* c; uint8_t* o; cudaMalloc(&c, 8); cudaMalloc(&o, 8);
  for (int v = 0; v < 3; ++v) {
    k<<<1, 32>>>(mo, ml, off, M, c, o, v);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %.1f cycles/match\n", v, (double)h / M);
  }
}
