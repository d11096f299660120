// kernels.h — host-visible launch wrappers of kernels.cu (internal).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pcp_internal.h"

namespace pcp {

// One CRC work unit: `len` payload bytes at absolute `start`, which end
// `after` bytes before the end of page `page`'s payload.
struct CrcWindow {
  uint64_t start;
  uint64_t len;
  uint64_t after;
  uint32_t page;
  uint32_t pad;
};

void upload_x2n(cudaStream_t st);
void build_shift_table(uint32_t* h_tab);  // kShiftTabWords entries
size_t cloud_smem_fixed();
cudaError_t set_cloud_smem(size_t bytes);
cudaError_t launch_crc_windows(const uint8_t* bytes, const CrcWindow* win, uint32_t n_win,
                               const uint32_t* shift_tab, uint32_t* acc, int sms,
                               cudaStream_t st);
cudaError_t launch_page_decode(const uint8_t* bytes, uint8_t* raw, const PageRef* pages,
                               const uint32_t* todo, const uint64_t* scratch_off,
                               uint8_t* scratch, uint32_t n_todo, int32_t* status,
                               cudaStream_t st, long long* timing = nullptr,
                               uint32_t* pj_ptr = nullptr, uint32_t* pj_changed = nullptr,
                               uint32_t pj_rounds = 0, uint8_t* pj_flags = nullptr,
                               uint32_t pj_split = 64);  // pj_ptr: phase 4 by pointer jumping
uint64_t lz4_scratch_bytes(uint64_t pay);  // per LZ4 page
// scalar parse → cloud interpreter → page verdicts → sample status
// grid_pre: the prefix launch of a split chain (a.split_at > 0), one CTA per cloud
// vx (optional): the multi-CTA voxel stage between a decode-only k_cloud
// launch into handoff_a and the rest of the chain.
struct VxArgs;
cudaError_t launch_wave(const WaveArgs& a, int grid, int grid_pre, int threads, size_t smem, cudaStream_t st,
                        cudaEvent_t k0, cudaEvent_t k1, const VxArgs* vx, uint32_t vx_tiles,
                        uint32_t vx_btiles, int sms, cudaEvent_t v0, cudaEvent_t v1, uint8_t* handoff_a);
cudaError_t occupancy_cloud(int* n, int threads, size_t smem, int min_blocks);
// Max co-resident clusters of `cluster` CTAs (k_cloud<1>, or k_apply_set).
cudaError_t occupancy_cloud_clusters(int* n, int threads, size_t smem, uint32_t cluster, bool apply);
cudaError_t set_apply_smem(size_t bytes);
// n bytes (rounded up to 16) from device memory into mapped pinned host memory.
cudaError_t launch_store_host(const uint8_t* src, uint8_t* dst_mapped, uint64_t n, cudaStream_t st);
// Per-wave CSR of variable-length batch fields (k_wave_offsets + k_compact_wave).
struct WaveCsr {
  uint32_t n_out, n_var;
  uint64_t stride[16];
  int32_t var_index[16];  // batch field -> varlen slot, or -1
  int32_t var_field[16];  // varlen slot -> batch field
  const uint8_t* outs[16];
  uint8_t* compact[16];
  uint64_t* woff;  // [n_var][n+1]
  uint32_t* dense; // [n_out]
};
cudaError_t launch_wave_csr(const uint64_t* out_len, const WaveCsr& c, uint32_t n, int sms,
                            cudaStream_t st);

cudaError_t launch_apply_set(const WaveArgs& a, int grid, int threads, size_t smem,
                             cudaStream_t st);
cudaError_t launch_crc_ranges(const uint8_t* bytes, const uint64_t* off, const uint64_t* len,
                              uint32_t n, const uint32_t* shift_tab, uint32_t* out,
                              cudaStream_t st);
cudaError_t launch_decode_pages(const uint8_t* bytes, const uint64_t* page_off, uint32_t n,
                                uint8_t* out, const uint64_t* out_off, const uint32_t* col_first,
                                const uint64_t* col_off, const uint64_t* col_len,
                                const uint32_t* shift_tab, const uint64_t* scratch_off,
                                uint8_t* scratch, int32_t* status, cudaStream_t st);

constexpr uint32_t kShiftEntries = 8192;
constexpr uint32_t kShiftTabWords = kShiftEntries + 3 * 1024;  // + stride multiplication tables (device_crc.cuh)

}  // namespace pcp
