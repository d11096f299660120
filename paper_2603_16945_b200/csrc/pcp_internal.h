// pcp_internal.h — types shared by the host runtime and the sm_100a kernels.
//
// Naming follows the reference domain (pages, groups, slices, samples,
// fields); see DESIGN.md §2 for the HBM layout these structs describe.
#pragma once

#include <cstddef>
#include <cstdint>

namespace pcp {

// Errc + 1 (errors.hpp:8-53); identical values to PCP_E_* in pcpipe_b200.h.
enum Status : int32_t {
  kOk = 0,
  kBadAlignment = 4,
  kColumnOutOfRange = 5,
  kChecksumMismatch = 6,
  kCorruptPage = 7,
  kSchemaMismatch = 8,
  kIoFailure = 9,
  kEmptyDataset = 10,
  kBadMagic = 11,
  kUnsupportedVersion = 12,
  kCorruptHeader = 13,
  kRangeOutOfBounds = 14,
  kSchemaConflict = 15,
  kOutOfRange = 16,
  kNotPadded = 17,
  kShutdown = 23,
  kMissingField = 24,
  kEmptyCloud = 25,
  kUnknownOp = 26,
  kOutOfBounds = 27,
  kWorkerPanic = 28,
  kShapeMismatch = 29,
};

// Page flags (format.hpp:69-71).
constexpr uint8_t kFlagOuterLz4 = 1;
constexpr uint8_t kFlagInnerDelta = 2;
constexpr uint8_t kFlagStoredRaw = 4;
constexpr uint32_t kPageHeaderBytes = 21;  // format.cpp:276-287

// Map kinds: reference order (transforms.hpp:10-20) + App. C extensions.
enum MapKind : int32_t {
  kNormalize = 0,
  kTranslate,
  kJitter,
  kRotate,
  kRandomScale,
  kFlipYz,
  kColorAugment,
  kRandomCrop,
  kDownsample,
  kFps = 16,
  kVoxel,
  kRangeCrop,
};

// Field kinds (format.hpp:25).
enum FieldKind : int32_t { kBytes = 0, kInt32, kInt64, kFloat32, kFloat64, kString };

constexpr int kMaxFields = 16;      // schema fields
constexpr int kMaxBytesFields = 8;  // bytes fields per sample
constexpr uint32_t kFpsRegPts = 20;  // FPS points per thread held in registers (kernels.cu)
constexpr uint32_t kFpsMailBytes = 2 * 128 * 32;  // cluster-FPS mailbox: [parity][<= 8 x 16 warps] x 32 B
// voxel sort scratch (u32): hist[8 passes][256] + wcnt[16 warps][256] + base[2][256]
constexpr uint32_t kSortScratchBytes = (8 * 256 + 16 * 256 + 2 * 256) * 4;
constexpr int kMaxOps = 16;         // map transforms per pipeline

// One serialized EncodedPage used by a wave (absolute offsets into the
// device byte store).  Parsed from the 21-byte page header at open time.
struct PageRef {
  uint64_t off;       // page start (header) in the byte store
  uint64_t raw_len;   // decoded length
  uint64_t pay_len;   // payload length
  uint64_t raw_dst;   // decode target offset in the wave raw arena, or ~0
  uint32_t crc;       // stored CRC-32 of the payload
  uint32_t flags;     // page flags
  uint32_t crc_mode;  // 0: standalone CRC kernel, 1: fused into the cloud kernel
  uint32_t n_cols;    // inner-delta columns (block pages; raw-page coords)
  uint64_t col_first; // first column in the wave column table
};

// Scalar-record parse result per sample row (format.cpp:379-474).
struct ScalarRec {
  uint64_t blob_start, blob_end;
  uint64_t lens[kMaxBytesFields];
  uint32_t n_lens;
  uint32_t vals_off;  // byte offset of this row's non-bytes values in the
                      // wave's value arena (schema order, packed)
  uint32_t vals_len;
  int32_t status;
};

// One sample of a wave.
struct SampleWork {
  uint64_t epoch, index;     // seed coordinates (Item, pipeline.cpp:447-448)
  uint64_t blob_start, blob_end;  // header blob range (MetadataEntry.sample_meta)
  uint32_t block_page;       // wave page index of the group's block page
  uint32_t scalar_page;      // wave page index of the group's scalar page
  uint32_t row;              // row inside the group
  uint32_t group;            // wave group index
};

// Wave group: the scalar page to parse and where its records land.
struct GroupWork {
  uint32_t scalar_page;
  uint32_t first_rec;  // wave ScalarRec index of row 0
  uint32_t n_rows;
  uint32_t vals_base;  // value-arena byte offset for row 0
};

struct OpDesc {
  int32_t kind;
  uint32_t seed_op_id;
  int32_t has_theta;
  float theta;
  int64_t num_points;
  uint32_t gather_mask;  // bytes-field bits moved by index ops (extension)
  int32_t counts;        // voxel: emit counts
  float voxel;
  int32_t has_origin;
  float origin[3];
  float lo[3], hi[3];
};

struct FieldDesc {
  int32_t kind;         // FieldKind
  uint32_t elems;       // element count (product of shape; 1 for scalars)
  int32_t bytes_index;  // index among bytes fields, -1 otherwise
  int32_t out_index;    // output slot (std::map name order)
};

// Per-cloud state of the multi-CTA voxel stage (voxel_wave.cu).
struct VxCloud {
  uint32_t n;          // input points (data)
  uint32_t n_tiles;    // tiles of the input / of the sorted words
  uint32_t tile0;      // first global tile of this cloud
  uint32_t kept;       // points surviving the range crop (all when none)
  uint64_t word0;      // first sort word of this cloud
  int32_t status;      // Errc+1 of the vx ops (0 OK)
  int32_t fail_op;     // 1-based failing op
  uint32_t fallback;   // 1: keys too wide for the packed sort -> k_cloud runs the ops
  uint32_t active;     // 1: the vx kernels process this cloud
  uint32_t mn[3], mx[3];  // ordered-float min / max per axis over kept points
  uint32_t nan;        // a kept point has a NaN coordinate
  float o[3];          // voxel origin
  uint32_t q0[3];      // smallest key per axis (subtracted: order-preserving)
  uint32_t bx[3];      // key bits per axis
  uint32_t kb, ib;     // key bits, point-index bits (word = key << ib | index)
  uint32_t passes;     // 8-bit radix passes
  uint32_t V;          // voxels
  // bucket (MSD) mode: stable scatter by the top key bits into buckets,
  // then every work item (whole buckets, <= kVxItemCap records) is sorted,
  // segmented and reduced in shared memory
  uint32_t msd;        // 1: bucket mode, 0: global LSD radix sort
  uint32_t btile0, n_btiles;  // scatter tiles (kVxBTile points)
  uint32_t bb, lowbits;       // bucket bits (<= 12), key bits below the bucket
  uint32_t n_items;           // work items
  uint32_t max_bucket;        // records in the largest bucket
  uint32_t hist[8][256];  // digit histogram per pass (whole cloud)
};

// Everything a wave launch needs (passed by value to the kernels).
struct WaveArgs {
  const uint8_t* bytes;     // device byte store (slice data areas)
  uint8_t* raw;             // wave raw arena (decoded LZ4 / scalar pages)
  const PageRef* pages;
  uint32_t n_pages;
  const uint64_t* col_off;  // inner-delta column table
  const uint64_t* col_len;
  const GroupWork* groups;
  uint32_t n_groups;
  const SampleWork* samples;
  uint32_t n_samples;
  ScalarRec* recs;
  uint8_t* vals;            // non-bytes values per row
  uint32_t* page_crc_acc;   // XOR accumulators (fused CRC)
  int32_t* page_status;     // per page
  int32_t* sample_status;   // per sample (Errc+1)
  int32_t* sample_op;       // failing op id per sample
  // schema
  int32_t n_fields;
  FieldDesc fields[kMaxFields];
  int32_t n_bytes_fields;
  int32_t role_data, role_normal, role_color, role_intensity;  // bytes index or -1
  uint32_t tracked_mask;    // bytes fields held as per-point buffers
  // ops
  int32_t n_ops;
  OpDesc ops[kMaxOps];
  uint64_t base_seed;
  // MT19937-64 states seeded ahead of k_cloud by k_seed_states, one per
  // (sample, RNG op): [n_samples][n_rng][312] words; rng_slot[k] = op k's
  // index among the RNG ops or -1.  mt_pre = nullptr: ops seed in k_cloud.
  uint64_t* mt_pre;
  int32_t n_rng;
  int8_t rng_slot[kMaxOps];
  // outputs: per output field, a slot of out_stride[f] bytes per sample
  int32_t n_out;
  uint8_t* out[kMaxFields];
  uint64_t out_stride[kMaxFields];
  uint64_t* out_len;        // [n_out][n_samples]
  int32_t bytes_out[kMaxBytesFields];  // output index of bytes field f (-1: dropped)
  uint32_t field_cap[kMaxBytesFields]; // tracked field f: max bytes per point
  int32_t* sample_where;    // 0 op/record, 1 scalar page, 2 block page
  const uint32_t* shift_tab;  // CRC chunk shifts (device_crc.cuh)
  // per-CTA placement
  uint32_t cap_points;      // max points any tracked buffer must hold
  uint32_t max_blob;        // max blob bytes (staging)
  int32_t smem_mode;        // 1: some per-CTA buffers live in shared memory
  // per-CTA buffer plan (host: plan_buffers): 0 staging, 1..4 index arrays,
  // 5..12 cur per bytes field, 13..20 alt per bytes field, 21/22 voxel keys,
  // 23 voxel counts, 24 cluster-FPS slice + mailbox, 25 voxel sort scratch
  // (digit histograms + per-warp counts).  Bytes (0 = absent) and
  // shared-memory placement bits.
  uint64_t buf_bytes[26];
  uint32_t buf_smem_mask;
  int32_t min_blocks;       // k_cloud instantiation: 1 (128 regs) or 2 (64 regs)
  uint8_t* gscratch;        // global scratch (smem_mode 0), per CTA
  uint64_t gscratch_per_cta;
  uint32_t force_serial_fy; // test hook: take the serial Fisher-Yates path
  float neg_zero;           // -0.0f, opaque to ptxas (FPS paired squares, kernels.cu)
  uint32_t fps_cluster;     // CTAs per cloud (thread-block cluster) for large-cloud FPS; 1 = none
  uint32_t fps_slice_pts;   // points per CTA slice in cluster FPS (buffer 24 sizing)
  unsigned long long* op_cycles;  // PCP_OP_TIMING: [0] stage+decode, [1..n_ops] ops, [n_ops+1] writes
  // chain split for cluster FPS: ops [0, split_at) run in a
  // one-CTA-per-cloud launch that hands the cloud to the cluster launch
  // through a per-sample buffer; split_at = 0: no split
  int32_t split_at;
  int32_t op_begin, op_end;       // this launch's op range
  // hand-off slots [n_samples][handoff_stride]: handoff_in = read the cloud
  // before op_begin (instead of decoding its page), handoff_out = write it
  // after op_end (instead of the batch slots); null = not used
  uint8_t* handoff_in;
  uint8_t* handoff_out;
  uint64_t handoff_stride;
  uint64_t handoff_off[kMaxBytesFields + 1];  // per tracked field, [kMaxBytesFields] = counts
  // multi-CTA voxel stage (voxel_wave.cu) for large clouds: ops
  // [vx_first, vx_last] ([range_crop,] voxel) run across the GPU between the
  // decode-only launch and the rest of the chain; vx_first = -1: none.
  // Clouds flagged `fallback` (keys too wide for the packed sort) run those
  // ops in k_cloud from their decoded slot (handoff_fallback).
  int32_t vx_first, vx_last;
  const VxCloud* vx_state;  // [n_samples]
  uint8_t* handoff_fallback;
  // cloud-set mode (pcp_apply_map): clouds come from CSR arrays instead of
  // pages; bytes-field slots 0..7 = data, normal, color, intensity, extra0..3
  int32_t set_mode;
  const uint64_t* set_offset;            // [n_samples + 1] points
  const uint8_t* set_src[kMaxBytesFields];
  const uint64_t* set_seeds;             // [n_samples]
  uint8_t* set_out[kMaxBytesFields];     // [n_samples][cap_points * elem]
  uint32_t set_elem[kMaxBytesFields];
  uint32_t* set_count;                   // [n_samples]
  uint32_t set_out_cap;                  // output slot capacity (points)
  // voxel / grid subsample
  int32_t voxel_scratch;    // carve u64 sort keys (2 x cap) + counts (cap)
  int32_t count_out;        // output index of the synthesized "count" field, -1 none
  int32_t* set_voxel_count; // pcp_apply_map: [n_samples][set_out_cap]
};

}  // namespace pcp
