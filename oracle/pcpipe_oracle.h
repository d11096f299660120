/* pcpipe_oracle.h — TEST INFRASTRUCTURE ONLY (the CPU oracle).
 *
 * Plain-C restatement of the reference hot path (arXiv 2603.16945 "pcpipe",
 * /root/reference/proj/core/src) plus the App. C definitions of the operators
 * the reference lacks (FPS, voxel/grid subsample, range crop, per-point field
 * gather).  Used only by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg, as the checker.  Never linked by the product library.
 *
 * Parity pinning: every reference-backed function here is checked against the
 * reference itself (oracle/_ref/libpcpipe_ref.so, built from the unmodified
 * sources) in tests/test_oracle.py.  FPS / voxel / range crop have no
 * reference: their definitions are pinned
 * by known-answer tests only ("parity pinned by definition").
 *
 * Status codes: 0 = OK, otherwise (int)Errc + 1 (errors.hpp:8-53).
 */
#ifndef PCPIPE_ORACLE_H
#define PCPIPE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Errc + 1, errors.hpp:8-53 (subset used here) */
enum {
  ORC_OK = 0,
  ORC_BAD_ALIGNMENT = 4,
  ORC_COLUMN_OUT_OF_RANGE = 5,
  ORC_CHECKSUM_MISMATCH = 6,
  ORC_CORRUPT_PAGE = 7,
  ORC_SCHEMA_MISMATCH = 8,
  ORC_MISSING_FIELD = 24,
  ORC_EMPTY_CLOUD = 25,
  ORC_UNKNOWN_OP = 26,
  ORC_OUT_OF_BOUNDS = 27,
};

/* ---- codec ------------------------------------------------------------ */
uint32_t orc_crc32(const uint8_t* p, size_t n);
int orc_lz4_decompress(const uint8_t* src, size_t n, uint8_t* dst, size_t raw_len);
int orc_xor_delta_decode(uint8_t* buf, size_t n, uint32_t width);
/* page = serialized EncodedPage; cols = (offset,length) pairs, width 4 */
int orc_decode_page(const uint8_t* page, size_t n, const uint64_t* col_off,
                    const uint64_t* col_len, size_t ncols, uint8_t* out,
                    size_t out_cap, size_t* out_len);

/* ---- RNG (libstdc++-13 restatement) ------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;
void orc_mt_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt_next(orc_mt64* g);
float orc_canonical(orc_mt64* g);
float orc_uniform_real(orc_mt64* g, float a, float b);
typedef struct {
  int saved_available;
  float saved;
} orc_normal;
float orc_normal_draw(orc_normal* d, orc_mt64* g, float mean, float stddev);
uint64_t orc_uniform_int(orc_mt64* g, uint64_t a, uint64_t b);
uint64_t orc_mix_seed(uint64_t base, uint64_t epoch, uint64_t index, uint64_t op);

/* ---- operators --------------------------------------------------------- */
enum {
  ORC_NORMALIZE = 0,
  ORC_TRANSLATE,
  ORC_JITTER,
  ORC_ROTATE,
  ORC_RANDOM_SCALE,
  ORC_FLIP_YZ,
  ORC_COLOR_AUGMENT,
  ORC_RANDOM_CROP,
  ORC_DOWNSAMPLE,
  /* extensions (no reference) */
  ORC_FPS = 16,
  ORC_VOXEL,
  ORC_RANGE_CROP,
};

#define ORC_MAX_EXTRA 4
typedef struct {
  /* per-point fields; NULL = absent.  Arrays hold cap points. */
  float* data;      /* [n][3] */
  float* normal;    /* [n_normal][3] */
  float* color;     /* [n_color][3] */
  float* intensity; /* [n_intensity] */
  size_t n, n_normal, n_color, n_intensity;
  /* extra per-point fields gathered by index ops when listed in "gather" */
  uint8_t* extra[ORC_MAX_EXTRA];
  size_t extra_elem[ORC_MAX_EXTRA]; /* bytes per point */
  size_t n_extra[ORC_MAX_EXTRA];    /* points */
  int32_t* counts;                  /* voxel counts out (cap) or NULL */
  size_t n_counts;
  size_t cap;
} orc_cloud;

typedef struct {
  int has_theta;
  float theta;
  int64_t num_points;
  int gather_intensity; /* downsample: also gather intensity (extension) */
  int gather_extra;     /* index ops gather extra[] too (extension) */
  float voxel_size;
  int has_origin;
  float origin[3];
  float lo[3], hi[3];
} orc_params;

int orc_apply_map(int kind, const orc_params* params, orc_cloud* c, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
