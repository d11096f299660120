// Calibration: cycles per dependent shared-memory load (pointer chase) for
// one thread, and for the walker pattern (load, mask, add, store tokpos).
#include <cstdio>
#include <cstdint>
__global__ void chase(uint32_t* out, long long* cyc, int steps, uint32_t* gout) {
  __shared__ uint32_t tab[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = (i * 97 + 13) & 2047;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t p = 0;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) p = tab[p];
    long long t1 = clock64();
    uint32_t q = 0, cnt = 0, pos = 0;
    for (int s = 0; s < steps; ++s) {
      const uint32_t v = tab[q];
      if (v & 0x80000000u) break;
      gout[cnt++ & 0xffff] = pos;
      pos += v & 0x3fffffffu;
      q = (q + v) & 2047;
    }
    long long t2 = clock64();
    __shared__ uint32_t sbuf[4096];
    uint32_t q2 = 0, cnt2 = 0, pos2 = 0, bad = 0;
    for (int s = 0; s < steps; ++s) {
      const uint32_t v = tab[q2];
      bad |= v;
      sbuf[cnt2++ & 4095] = pos2;
      pos2 += v & 0x3fffffffu;
      q2 = (q2 + v) & 2047;
    }
    long long t3 = clock64();
    out[0] = p + pos + cnt + pos2 + bad + sbuf[5];
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
}
int main() {
  uint32_t *o, *g;
  long long* c;
  cudaMalloc(&o, 4);
  cudaMalloc(&g, 65536 * 4);
  cudaMalloc(&c, 24);
  const int steps = 100000;
  chase<<<1, 128>>>(o, c, steps, g);
  long long h[3];
  cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("pure chase %.1f, walker+STG %.1f, walker+STS %.1f cycles/step\n", (double)h[0] / steps,
         (double)h[1] / steps, (double)h[2] / steps);
}
