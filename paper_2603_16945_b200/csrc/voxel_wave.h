// voxel_wave.h — multi-CTA voxel / grid subsample stage (voxel_wave.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pcp_internal.h"

namespace pcp {

constexpr uint32_t kVxMaxPasses = 6;  // 8-bit digits: keys up to 48 bits (wider: k_cloud fallback)
constexpr uint32_t kVxMaxBucketBits = 20;  // bucket mode: up to 20 top key bits (1 Mi buckets)
constexpr uint32_t kVxSmemBuckets = 4096;  // histograms / ranks in shared memory up to this many
constexpr uint32_t kVxMaxPayWords = 8;     // staged payload per record (32 B): else read from B
constexpr uint32_t kVxBTile = 4096;    // bucket mode: points per scatter tile
constexpr uint32_t kVxItemCap = 2048;  // bucket mode: records per work item (shared memory)

// Arguments of the stage (by value).  A = decoded clouds (hand-off slots of
// the decode-only k_cloud launch), voxelized in place by the stage (the rest
// of the chain reads A); B = scratch slots of the same layout (the sorted
// payload); both [n_samples][stride] with the k_cloud hand-off header and
// field offsets `off`.
struct VxArgs {
  uint32_t n_samples;
  uint8_t* A;
  uint8_t* B;
  uint64_t stride;
  uint64_t off[kMaxBytesFields + 1];
  int32_t n_bytes_fields;
  int32_t role_data, role_normal, role_color, role_intensity;
  uint32_t mm;          // fields the ops move (roles + gathered extras)
  int32_t has_crop;     // leading range_crop (vx_first) before the voxel op (vx_last)
  float lo[3], hi[3];
  float voxel;
  int32_t has_origin;
  float origin[3];
  int32_t counts;       // emit per-voxel counts
  int32_t vx_first, vx_last;
  uint32_t max_passes;  // radix passes launched (kernels skip passes a cloud does not need)
  // scratch
  VxCloud* cl;          // [n_samples]
  uint32_t* total_tiles;
  uint32_t* tile_cloud;  // [tiles]
  uint32_t* tile_kept;   // [tiles] kept points, later voxel starts
  uint32_t* tile_kofs;   // [tiles] compaction offsets, later voxel offsets
  uint32_t* cnt;         // [tiles][256]
  uint64_t* w0;          // [points] sort words (ping)
  uint64_t* w1;          // (pong)
  uint64_t* w2;          // [2 x points] bucket mode: sort buffers of dense items
  // bucket mode scratch
  uint32_t* total_btiles;
  uint32_t* btile_cloud;  // [btiles]
  uint32_t bucket_bits;   // per-cloud bucket bits cap (<= kVxMaxBucketBits)
  uint32_t bstride;       // 1 << bucket_bits
  uint32_t pay_words;     // staged payload words per record (0: not staged)
  uint32_t* bcur;         // [n_samples][bstride]: bucket write cursors
  uint32_t* boff;         // [n_samples][bstride + 4]: bucket totals -> offsets (+ total)
  uint32_t* any_lsd;      // a cloud of the wave takes the global LSD sort
  uint32_t* item_v;       // [n_samples][max_items]: voxels per item -> voxel offsets
  uint32_t* item_b;       // [n_samples][max_items]: first bucket of each item
  uint32_t max_items;
  uint8_t* T;             // voxel results per item before compaction (slots like A)
  int32_t msd_enabled;    // 0: every cloud takes the LSD path
  // statuses of failing clouds (the rest report from the last k_cloud launch)
  int32_t* sample_status;
  int32_t* sample_op;
  int32_t* sample_where;
};

// tiles_bound: an upper bound of the wave's tiles (sum over samples of
// ceil(points / voxel_wave_tile_points())).
cudaError_t launch_voxel_wave(const VxArgs& v, uint32_t tiles_bound, uint32_t btiles_bound, int sms,
                              cudaStream_t st);
// Dynamic shared memory of the bucket-mode item kernel.
size_t voxel_wave_item_smem(uint32_t pay_words);
uint32_t voxel_wave_tile_points();

}  // namespace pcp
