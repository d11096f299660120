/* pcpipe_b200.h — C ABI of the B200-native PcRecord → training-batch stage.
 *
 * Drop-in for the hot path of the reference library "pcpipe"
 * (arXiv 2603.16945; reference sources under proj/core/ of the reference
 * tree).  Each entry point names the reference interface it replaces.
 *
 *   - plain pointers and sizes only; no CUDA/torch types in signatures
 *     (`stream` is a cudaStream_t passed as void*, NULL = the legacy stream);
 *   - every call returns an int status: 0 = OK, otherwise (int)Errc + 1 with
 *     Errc exactly as errors.hpp:8-53 (PCP_E_* below); pcp_last_error() holds
 *     the message (thread-local).  No C++ exception crosses this ABI;
 *   - device-side failures (CRC mismatch, corrupt LZ4, blob overrun, empty
 *     cloud …) surface at the batch boundary as PCP_E_WORKER_PANIC naming the
 *     op, exactly like Pipeline::next_batch (pipeline.cpp:677-689).
 *
 * There is no CPU fallback: on a host without a usable sm_100 device every
 * compute entry point returns PCP_E_IO_FAILURE with a message saying so.
 */
#ifndef PCPIPE_B200_H
#define PCPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes = (int)pcpipe::Errc + 1 (errors.hpp:8-53) ---------- */
enum {
  PCP_OK = 0,
  PCP_E_DUPLICATE_FIELD = 1,
  PCP_E_EMPTY_SCHEMA,
  PCP_E_BAD_SHAPE,
  PCP_E_BAD_ALIGNMENT,
  PCP_E_COLUMN_OUT_OF_RANGE,
  PCP_E_CHECKSUM_MISMATCH,
  PCP_E_CORRUPT_PAGE,
  PCP_E_SCHEMA_MISMATCH,
  PCP_E_IO_FAILURE,
  PCP_E_EMPTY_DATASET,
  PCP_E_BAD_MAGIC,
  PCP_E_UNSUPPORTED_VERSION,
  PCP_E_CORRUPT_HEADER,
  PCP_E_RANGE_OUT_OF_BOUNDS,
  PCP_E_SCHEMA_CONFLICT,
  PCP_E_OUT_OF_RANGE,
  PCP_E_NOT_PADDED,
  PCP_E_MALFORMED_HEADER,
  PCP_E_TRUNCATED_PAYLOAD,
  PCP_E_UNSUPPORTED_PROPERTY,
  PCP_E_NO_INPUT_FILES,
  PCP_E_PARSE_FAILURE,
  PCP_E_SHUTDOWN,
  PCP_E_MISSING_FIELD,
  PCP_E_EMPTY_CLOUD,
  PCP_E_UNKNOWN_OP,
  PCP_E_OUT_OF_BOUNDS,
  PCP_E_WORKER_PANIC,
  PCP_E_SHAPE_MISMATCH,
};

/* Thread-local message of the last failing call on this thread. */
const char* pcp_last_error(void);
/* Errc name for a status ("kChecksumMismatch" …), errors.cpp:5-50. */
const char* pcp_errc_name(int status);
/* Library/device info; returns PCP_OK when an sm_100 device is usable. */
int pcp_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);

/* ---- seeding: mix_seed (transforms.hpp:27-28, transforms.cpp:82-96) --- */
uint64_t pcp_mix_seed(uint64_t base_seed, uint64_t epoch, uint64_t sample_index,
                      uint64_t op_id);

/* ---- codec (format.hpp:88-105, lz4_block.hpp:22-26) -------------------
 * Batched page decode on the device.  d_bytes holds serialized EncodedPage
 * records ([u8 flags][u64 raw_len][u64 payload_len][u32 crc][payload],
 * format.cpp:276-299) at d_page_off[i]; each decodes to d_out + d_out_off[i]
 * (capacity raw_len).  Inner-delta columns (offset,length pairs in raw-page
 * coordinates, width 4) are d_col_off/d_col_len[d_col_first[i] ..
 * d_col_first[i+1]).  Per-page status (0 or Errc+1: kChecksumMismatch,
 * kCorruptPage, kColumnOutOfRange, kBadAlignment) lands in d_status[i].
 * Replaces decode_block_page / decode_scalar_page (format.cpp:243-274). */
int pcp_decode_pages(const uint8_t* d_bytes, const uint64_t* d_page_off, uint32_t n_pages,
                     uint8_t* d_out, const uint64_t* d_out_off,
                     const uint32_t* d_col_first, const uint64_t* d_col_off,
                     const uint64_t* d_col_len, int32_t* d_status, void* stream);

/* zlib-compatible CRC-32 of n_ranges byte ranges of device memory
 * (crc32_of, format.cpp:163-166).  Results to d_crc[i]. */
int pcp_crc32_ranges(const uint8_t* d_bytes, const uint64_t* d_off, const uint64_t* d_len,
                     uint32_t n_ranges, uint32_t* d_crc, void* stream);

/* ---- operators: apply_map (transforms.hpp:33-34) over a cloud set -----
 * A cloud set is CSR over n_clouds clouds in device memory.  Per-point
 * fields are optional (NULL = absent): data/normal/color float32 [N][3],
 * intensity float32 [N], plus up to 4 extra per-point byte fields gathered
 * by index ops when listed in params "gather".  apply_map semantics per cloud
 * c with seed d_seeds[c]; outputs go to `out` (capacity out->cap_points per
 * cloud, dense slots of that stride; out->d_count receives sizes).
 * kind: PCP_MAP_* (map_kind_from_name names, transforms.cpp:54-80, plus the
 * App. C extensions).  Per-cloud status → d_status[c]. */
enum {
  PCP_MAP_NORMALIZE = 0,
  PCP_MAP_TRANSLATE,
  PCP_MAP_JITTER,
  PCP_MAP_ROTATE,
  PCP_MAP_RANDOM_SCALE,
  PCP_MAP_FLIP_YZ,
  PCP_MAP_COLOR_AUGMENT,
  PCP_MAP_RANDOM_CROP,
  PCP_MAP_DOWNSAMPLE,
  PCP_MAP_FPS = 16,
  PCP_MAP_VOXEL,
  PCP_MAP_RANGE_CROP,
};
int pcp_map_kind_from_name(const char* name, int* kind);

typedef struct {
  uint32_t n_clouds;
  const uint64_t* d_offset; /* input: [n_clouds+1] point offsets (CSR) */
  float* d_data;            /* [total][3] (required) */
  float* d_normal;          /* [total][3] or NULL */
  float* d_color;           /* [total][3] or NULL */
  float* d_intensity;       /* [total] or NULL */
  uint8_t* d_extra[4];      /* [total][extra_elem[e]] or NULL */
  uint32_t extra_elem[4];
} pcp_cloud_set;

typedef struct {
  uint32_t cap_points; /* per-cloud slot capacity */
  float* d_data;       /* [n_clouds][cap][3] */
  float* d_normal;
  float* d_color;
  float* d_intensity;
  uint8_t* d_extra[4];
  int32_t* d_voxel_count; /* [n_clouds][cap] (voxel only) or NULL */
  uint32_t* d_count;      /* [n_clouds] points out */
} pcp_cloud_out;

int pcp_apply_map(int kind, const char* params_json, const pcp_cloud_set* in,
                  const pcp_cloud_out* out, const uint64_t* d_seeds, int32_t* d_status,
                  void* stream);

/* ---- dataset writer (format.cpp:499-610), host side -------------------
 * Writes <out_dir>/<stem>.pcrecord[N] byte-identical to write_dataset.
 * schema_json = Schema::to_json ({"fields": {...}}).  samples = TLV stream
 * (u32 n_fields {u16 name_len, name, u8 kind, u64 nbytes, bytes}) * n. */
int pcp_write_dataset(const char* out_dir, const char* stem, const char* schema_json,
                      const uint8_t* samples_tlv, size_t tlv_len, uint32_t n_samples,
                      uint32_t slice_count, uint32_t group_size, uint32_t n_threads);
/* The same files with every page encoded on `device` (XOR-delta columns, the
 * reference's greedy LZ4 compressor, stored-raw fallback, payload CRC-32:
 * encode_block_page / encode_scalar_page, format.cpp:198-274, and
 * lz4::compress, lz4_block.cpp:33-103), byte-identical. */
int pcp_write_dataset_device(const char* out_dir, const char* stem, const char* schema_json,
                             const uint8_t* samples_tlv, size_t tlv_len, uint32_t n_samples,
                             uint32_t slice_count, uint32_t group_size, int device);

/* ---- pipeline (pipeline.hpp:157-186) -----------------------------------
 * Opens <primary>.pcrecord (+ continuation slices), parses the reference
 * graph JSON (PipelineGraph::from_json, pipeline.cpp:122-146) and runs
 * source → maps → batch on `device`.  entry_ids (optional) is the list of
 * index entries this pipeline walks — e.g. one GPU's shard; index i of the
 * walk is the seed index, like Item.index (pipeline.cpp:447-448).
 * Options: JSON {"epochs": n, "resident": true|false, "wave_batches": k,
 * "slots": s, "host_batches": true|false, "stream": true|false,
 * "reader_threads": t, "serial": true|false, "vx": true|false,
 * "lz4_pointer_jumping": true|false}.
 *   resident      pages of the walk's slices in HBM (read once at open);
 *                 false: in pinned host memory, H2D per wave
 *   stream        no copy at open: reader threads read each wave's pages from
 *                 the slice files into the wave slot's pinned buffer ahead
 *                 of its launch (datasets larger than host RAM / HBM)
 *   host_batches  every batch also in pinned host memory (pcp_field.h_ptr),
 *                 like the reference's host Batch: one D2H per field per wave
 *   serial        one wave in flight (non-overlapped per-kernel timing)
 *   vx            multi-CTA voxel stage for large clouds
 *   lz4_pointer_jumping  LZ4 match resolution over all pages of a wave at
 *                 once (default: unless the block pages average >= 32
 *                 samples) or one warp per page
 * Only the slices the walk touches are read (shard-local loading). */
typedef struct pcp_pipeline pcp_pipeline;

int pcp_pipeline_open(const char* primary_path, const char* graph_json,
                      const uint64_t* entry_ids, uint64_t n_entries, int device,
                      const char* options_json, pcp_pipeline** out);

/* Caller-supplied pages: the SourceFn analogue (Pipeline(graph, SourceFn,
 * samples_per_epoch, opts), pipeline.hpp:157-160; the streaming SourceFn of
 * stream_dataset, streaming.cpp:324-351, blocks until a sample's slice is
 * staged).  The stage asks `read` for byte ranges of slice data areas (offset
 * 0 = first byte after the primary slice's header; continuation slices from
 * their first byte), from reader threads, ahead of each wave; `read` may block
 * until the slice is present and returns 0 or an Errc+1 status (surfaced
 * from next_batch).  `done` (optional) is called on the caller's thread once
 * the pages of walk positions [first_index, first_index+count) of `epoch` are
 * on the device (their host bytes may be evicted).  `header` = the primary
 * slice's FileHeader bytes ("PCRC", version, JSON length, JSON), e.g. from a
 * meta index.  Options as pcp_pipeline_open ("stream" is implied). */
typedef int (*pcp_page_source_fn)(void* user, uint32_t slice, uint64_t offset, uint64_t length,
                                  uint8_t* dst);
typedef void (*pcp_wave_done_fn)(void* user, uint64_t epoch, uint64_t first_index, uint64_t count);
int pcp_pipeline_open_source(const uint8_t* header, size_t header_len, const char* graph_json,
                             const uint64_t* entry_ids, uint64_t n_entries, int device,
                             const char* options_json, pcp_page_source_fn read,
                             pcp_wave_done_fn done, void* user, pcp_pipeline** out);

#define PCP_MAX_BATCH_FIELDS 16
typedef struct {
  char name[48];
  int32_t kind;              /* 0 bytes 1 int32 2 int64 3 float32 4 float64 */
  uint8_t* d_ptr;            /* device, samples concatenated in order */
  uint64_t nbytes;           /* total bytes */
  const uint64_t* h_offsets; /* host [n_samples+1] byte offsets per sample */
  int32_t uniform;           /* 1 when every sample has the same length */
  const uint8_t* h_ptr;      /* option host_batches: the field in pinned host
                                memory (else NULL); d_ptr is then NULL for a
                                ragged field */
} pcp_field;

typedef struct {
  uint64_t epoch;
  uint64_t batch_index;
  uint32_t n_samples;
  uint32_t n_fields;
  pcp_field fields[PCP_MAX_BATCH_FIELDS]; /* std::map (name) order */
} pcp_batch;

/* Next batch in dataset order (Pipeline::next_batch); *end_of_stream = 1
 * and PCP_OK once the final epoch drained.
 * View lifetime: every pointer in *out (d_ptr, h_ptr, h_offsets) is valid
 * until the NEXT pcp_pipeline_next_batch / pcp_pipeline_close call on this
 * handle.  Device reads of d_ptr must be enqueued on pcp_pipeline_stream()
 * before that call: the slot is refilled only after the work already queued
 * on that stream (the reference returns Batch by value; copy what you keep).
 * Variable-length fields (crop / voxel outputs, strings) are CSR: d_ptr is
 * contiguous over the batch's samples with h_offsets[k] byte offsets. */
int pcp_pipeline_next_batch(pcp_pipeline* p, pcp_batch* out, int* end_of_stream);
/* Stream on which the returned batch views are ready (use it for D2H of the
 * batch; waves are computed on an internal stream). cudaStream_t as void*. */
void* pcp_pipeline_stream(pcp_pipeline* p);
/* Stats JSON (clouds, points, bytes, kernel ms …); caller must not free. */
const char* pcp_pipeline_stats(pcp_pipeline* p);
/* Pipeline::metrics (pipeline.hpp:140-149): MetricsSnapshot as JSON
 * {uptime_seconds, ops:[{op_id, kind, num_workers, items, busy_seconds,
 * out_queue_size, out_queue_capacity}], sink_polls, sink_empty_polls,
 * sink_size, sink_capacity, batches_emitted, items_emitted} plus the GPU
 * knobs (slots, wave_batches).  Valid until the next call; do not free. */
const char* pcp_pipeline_metrics(pcp_pipeline* p);
/* Pipeline::update_op_config (pipeline.hpp:168-170) for the device knobs:
 * JSON {"slots": 2..8, "wave_batches": k >= 1}.  Applied at the next wave
 * boundary after the waves in flight are served; batches, their order and
 * their seeds do not change.  PCP_E_OUT_OF_BOUNDS for values out of range
 * (or while streaming from files), PCP_E_UNKNOWN_OP for unknown knobs. */
int pcp_pipeline_update_config(pcp_pipeline* p, const char* config_json);
void pcp_pipeline_close(pcp_pipeline* p);

/* ---- small device-memory helpers for hosts without a CUDA runtime ----- */
int pcp_malloc(void** d_ptr, size_t n);
int pcp_free(void* d_ptr);
int pcp_memcpy_h2d(void* d_dst, const void* h_src, size_t n, void* stream);
int pcp_memcpy_d2h(void* h_dst, const void* d_src, size_t n, void* stream);
/* Asynchronous variant: enqueues the copy on `stream` (use the batch's
 * pcp_batch.stream / pcp_pipeline_stream) and returns; the data is in h_dst
 * after pcp_stream_sync(stream).  The pipeline will not reuse a batch's
 * device buffers before copies enqueued on its serve stream complete. */
int pcp_memcpy_d2h_async(void* h_dst, const void* d_src, size_t n, void* stream);
int pcp_stream_sync(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PCPIPE_B200_H */
