// Standalone micro-benchmark of the CTA-parallel LZ4 decoder on ONE page
// (diagnostics, not part of the library).  Usage: lz4_microbench <page.bin>
// where page.bin = [u32 raw_len][payload].  Prints per-phase clocks.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../paper_2603_16945_b200/csrc/lz4_parallel.cuh"

using namespace pcp;

__global__ void k(const uint8_t* src, uint32_t n, uint8_t* dst, uint32_t raw, uint8_t* scr,
                  long long* tm, int* st) {
  __shared__ __align__(16) uint32_t ctl[lz4p::kSmemWords];
  lz4p::Scratch sc = lz4p::carve_scratch(scr, n);
  int r = lz4p::decode_block(src, n, dst, raw, sc, ctl, tm);
  if (threadIdx.x == 0) *st = r;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  uint32_t raw;
  fread(&raw, 4, 1, f);
  std::vector<uint8_t> pay;
  uint8_t buf[65536];
  size_t k_;
  while ((k_ = fread(buf, 1, sizeof buf, f)) > 0) pay.insert(pay.end(), buf, buf + k_);
  fclose(f);
  uint8_t *d_src, *d_dst, *d_scr;
  long long* d_tm;
  int* d_st;
  cudaMalloc(&d_src, pay.size() + 64);
  cudaMalloc(&d_dst, raw + 64);
  cudaMalloc(&d_scr, lz4p::scratch_bytes(pay.size()));
  cudaMalloc(&d_tm, 8 * 8192);
  cudaMalloc(&d_st, 4);
  cudaMemcpy(d_src, pay.data(), pay.size(), cudaMemcpyHostToDevice);
  for (int it = 0; it < 3; ++it) {
    cudaMemset(d_tm, 0, 8 * 8192);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<1, 256>>>(d_src, (uint32_t)pay.size(), d_dst, raw, d_scr, d_tm, d_st);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long tm[16];
    int st;
    cudaMemcpy(tm, d_tm, 128, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, d_st, 4, cudaMemcpyDeviceToHost);
    printf("status %d  %.3f ms  skim %lld (walk %lld fill %lld)  phase3 %lld  matches %lld jump %lld (rounds %lld, span bytes %lld) waves %lld slow %lld\n",
           st, ms, tm[2] - tm[0], tm[8], tm[9], tm[3] - tm[2], tm[4] - tm[3], tm[7], tm[10], tm[11], tm[5], tm[6]);
  }
#ifdef PCP_EXP_TRACE
  {
    std::vector<long long> tr(4096);
    cudaMemcpy(tr.data(), d_tm, 8 * 4096, cudaMemcpyDeviceToHost);
    std::vector<long long> d;
    for (int w = 1; w < 900; ++w) d.push_back(tr[16 + w] - tr[15 + w]);
    std::vector<long long> srt = d;
    std::sort(srt.begin(), srt.end());
    long long sum = 0;
    for (auto x : d) sum += x;
    printf("window cycles: sum %lld median %lld p90 %lld p99 %lld max %lld\n", sum, srt[srt.size() / 2],
           srt[srt.size() * 9 / 10], srt[srt.size() * 99 / 100], srt.back());
    for (int w = 8; w < 32; ++w)
      printf("w%d: %lld cyc, tokens %lld, pos %lld (window start %d) steps2 %lld steps1 %lld specials %lld\n", w, tr[17 + w] - tr[16 + w],
             tr[1041 + w] - tr[1040 + w], tr[2064 + w], w * 2048, tr[3088 + w] & 0xFFFFF, (tr[3088 + w] >> 20) & 0xFFFFF, tr[3088 + w] >> 40);
  }
#endif
  std::vector<uint8_t> out(raw);
  cudaMemcpy(out.data(), d_dst, raw, cudaMemcpyDeviceToHost);
  FILE* o = fopen("/tmp/lz4_out.bin", "wb");
  fwrite(out.data(), 1, raw, o);
  fclose(o);
  return 0;
}
