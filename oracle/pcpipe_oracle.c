/* pcpipe_oracle.c — TEST INFRASTRUCTURE ONLY (the CPU oracle).
 *
 * Restatement of the reference hot path, function by function, each citing the
 * reference file:line it follows (paths under /root/reference/proj/core/).
 * Compiled with -ffp-contract=off, like the reference's x86-64 Release build
 * (no -march, hence no FMA), so float/double rounding follows the same
 * sequence of IEEE operations.  See pcpipe_oracle.h for the parity-pinning
 * story.  Not a product path: nothing under paper_2603_16945_b200/ links it.
 */
#define _GNU_SOURCE
#include "pcpipe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================== */
/* codec                                                                    */
/* ======================================================================== */

/* zlib crc32 (format.cpp:163-166 calls ::crc32(0, p, n)): reflected
 * polynomial 0xEDB88320, init 0xFFFFFFFF, final xor 0xFFFFFFFF. */
static uint32_t crc_table[256];
static int crc_ready = 0;

static void crc_init(void) {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    crc_table[i] = c;
  }
  crc_ready = 1;
}

uint32_t orc_crc32(const uint8_t* p, size_t n) {
  if (!crc_ready) crc_init();
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = crc_table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

/* lz4::decompress, lz4_block.cpp:113-156 — same checks in the same order. */
int orc_lz4_decompress(const uint8_t* src, size_t n, uint8_t* dst, size_t raw_len) {
  size_t ip = 0, op = 0;
  for (;;) {
    if (ip >= n) return ORC_CORRUPT_PAGE; /* truncated stream :134 */
    const uint8_t token = src[ip++];
    size_t lit = token >> 4;
    if (lit == 15) { /* read_len_ext :120-131 */
      uint8_t b;
      do {
        if (ip >= n) return ORC_CORRUPT_PAGE;
        b = src[ip++];
        lit += b;
      } while (b == 255);
    }
    if (ip + lit > n || op + lit > raw_len) return ORC_CORRUPT_PAGE; /* :137 */
    memcpy(dst + op, src + ip, lit);
    ip += lit;
    op += lit;
    if (ip == n) return op == raw_len ? ORC_OK : ORC_CORRUPT_PAGE; /* :141-144 */
    if (ip + 2 > n) return ORC_CORRUPT_PAGE;                       /* :145 */
    const size_t offset = (size_t)src[ip] | ((size_t)src[ip + 1] << 8);
    ip += 2;
    if (offset == 0 || offset > op) return ORC_CORRUPT_PAGE; /* :148 */
    size_t ml = token & 0x0f;
    if (ml == 15) {
      uint8_t b;
      do {
        if (ip >= n) return ORC_CORRUPT_PAGE;
        b = src[ip++];
        ml += b;
      } while (b == 255);
    }
    ml += 4;                                    /* kMinMatch :11 */
    if (op + ml > raw_len) return ORC_CORRUPT_PAGE; /* :150 */
    for (size_t i = 0; i < ml; ++i) dst[op + i] = dst[op - offset + i]; /* :151-153 */
    op += ml;
  }
}

/* xor_delta_decode, format.cpp:183-195: w[i] ^= w[i-1], in place. */
int orc_xor_delta_decode(uint8_t* buf, size_t n, uint32_t width) {
  if (width != 4 && width != 8) return ORC_BAD_ALIGNMENT;
  if (n % width) return ORC_BAD_ALIGNMENT;
  for (size_t i = width; i + width <= n; i += width)
    for (size_t b = 0; b < width; ++b) buf[i + b] ^= buf[i - width + b];
  return ORC_OK;
}

/* EncodedPage::deserialize (format.cpp:289-299) + decode_block_page
 * (format.cpp:243-266): [u8 flags][u64 raw_len][u64 payload_len][u32 crc]. */
int orc_decode_page(const uint8_t* page, size_t n, const uint64_t* col_off,
                    const uint64_t* col_len, size_t ncols, uint8_t* out,
                    size_t out_cap, size_t* out_len) {
  if (n < 21) return ORC_CORRUPT_PAGE;
  uint8_t flags = page[0];
  uint64_t raw_len, pay_len;
  uint32_t crc;
  memcpy(&raw_len, page + 1, 8);
  memcpy(&pay_len, page + 9, 8);
  memcpy(&crc, page + 17, 4);
  if (21 + pay_len > n) return ORC_CORRUPT_PAGE;
  const uint8_t* payload = page + 21;
  if (orc_crc32(payload, pay_len) != crc) return ORC_CHECKSUM_MISMATCH;
  if (raw_len > out_cap) return ORC_OUT_OF_BOUNDS;
  if (flags & 1) {
    int st = orc_lz4_decompress(payload, pay_len, out, raw_len);
    if (st) return st;
  } else if (flags & 4) {
    if (pay_len != raw_len) return ORC_CORRUPT_PAGE;
    memcpy(out, payload, raw_len);
  } else {
    return ORC_CORRUPT_PAGE;
  }
  if (flags & 2) { /* check_columns format.cpp:199-207 then per-column decode */
    for (size_t c = 0; c < ncols; ++c) {
      if (col_off[c] + col_len[c] > raw_len) return ORC_COLUMN_OUT_OF_RANGE;
      if (col_len[c] % 4) return ORC_BAD_ALIGNMENT;
    }
    for (size_t c = 0; c < ncols; ++c) orc_xor_delta_decode(out + col_off[c], col_len[c], 4);
  }
  *out_len = raw_len;
  return ORC_OK;
}

/* ======================================================================== */
/* RNG: libstdc++ 13 restatement                          */
/* ======================================================================== */

/* std::mt19937_64 seeding: x[i] = f*(x[i-1] ^ (x[i-1] >> 62)) + i */
void orc_mt_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static void mt_twist(orc_mt64* g) {
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  const uint64_t A = 0xB5026F5AA96619E9ull;
  for (int i = 0; i < 312; ++i) {
    uint64_t y = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
    g->mt[i] = g->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? A : 0);
  }
  g->idx = 0;
}

uint64_t orc_mt_next(orc_mt64* g) {
  if (g->idx >= 312) mt_twist(g);
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

/* generate_canonical<float,24> (random.tcc:3349-3381): one draw. */
float orc_canonical(orc_mt64* g) {
  float r = (float)orc_mt_next(g) / 18446744073709551616.0f;
  if (r >= 1.0f) r = nextafterf(1.0f, 0.0f);
  return r;
}

/* uniform_real_distribution<float>: canon * (b - a) + a (random.h:1909). */
float orc_uniform_real(orc_mt64* g, float a, float b) {
  float c = orc_canonical(g);
  float w = b - a;
  float m = c * w;
  return m + a;
}

/* normal_distribution<float> polar method (random.tcc:1811-1843). */
float orc_normal_draw(orc_normal* d, orc_mt64* g, float mean, float stddev) {
  float ret;
  if (d->saved_available) {
    d->saved_available = 0;
    ret = d->saved;
  } else {
    float x, y, r2;
    do {
      x = (float)((double)(2.0f * orc_canonical(g)) - 1.0);
      y = (float)((double)(2.0f * orc_canonical(g)) - 1.0);
      float xx = x * x, yy = y * y;
      r2 = xx + yy;
    } while (r2 > 1.0f || r2 == 0.0f);
    float lg = logf(r2);
    float num = -2.0f * lg;
    float q = num / r2;
    float mult = sqrtf(q);
    d->saved = x * mult;
    d->saved_available = 1;
    ret = y * mult;
  }
  float s = ret * stddev;
  return s + mean;
}

/* uniform_int_distribution<size_t>(a,b) with a 64-bit engine:
 * Lemire nearly-divisionless (uniform_int_dist.h _S_nd:257-281). */
uint64_t orc_uniform_int(orc_mt64* g, uint64_t a, uint64_t b) {
  const uint64_t urange = b - a;
  if (urange == UINT64_MAX) return orc_mt_next(g) + a;
  const uint64_t range = urange + 1;
  unsigned __int128 p = (unsigned __int128)orc_mt_next(g) * range;
  uint64_t low = (uint64_t)p;
  if (low < range) {
    uint64_t thr = (0 - range) % range;
    while (low < thr) {
      p = (unsigned __int128)orc_mt_next(g) * range;
      low = (uint64_t)p;
    }
  }
  return (uint64_t)(p >> 64) + a;
}

/* mix_seed, transforms.cpp:82-96 (splitmix64 chain). */
static uint64_t mix1(uint64_t h, uint64_t v) {
  h += 0x9e3779b97f4a7c15ull + v;
  h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
  h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
  return h ^ (h >> 31);
}
uint64_t orc_mix_seed(uint64_t base, uint64_t epoch, uint64_t index, uint64_t op) {
  uint64_t h = mix1(base, 0x706370ull);
  h = mix1(h, epoch);
  h = mix1(h, index);
  return mix1(h, op);
}

/* ======================================================================== */
/* operators (transforms.cpp:98-306) + App. C extensions                     */
/* ======================================================================== */

static float clampf_(float v, float lo, float hi) { /* std::clamp */
  return v < lo ? lo : (hi < v ? hi : v);
}

/* Gather every present per-point field by idx[0..m) (reference `take`/`filter`,
 * transforms.cpp:249-256,288-293).  Which fields move is decided by the caller
 * through the flags, mirroring the reference op's own choice. */
static void gather3(float* f, const size_t* idx, size_t m, float* tmp) {
  for (size_t i = 0; i < m; ++i) memcpy(tmp + 3 * i, f + 3 * idx[i], 12);
  memcpy(f, tmp, 12 * m);
}
static void gather1(float* f, const size_t* idx, size_t m, float* tmp) {
  for (size_t i = 0; i < m; ++i) tmp[i] = f[idx[i]];
  memcpy(f, tmp, 4 * m);
}
static void gatherb(uint8_t* f, size_t es, const size_t* idx, size_t m, uint8_t* tmp) {
  for (size_t i = 0; i < m; ++i) memcpy(tmp + es * i, f + es * idx[i], es);
  memcpy(f, tmp, es * m);
}

static int gather_all(orc_cloud* c, const size_t* idx, size_t m, int normals,
                      int colors, int intensity, int extra) {
  size_t need = m * 12 > 16 ? m * 12 : 16;
  for (int e = 0; e < ORC_MAX_EXTRA; ++e)
    if (c->extra[e] && c->extra_elem[e] * m > need) need = c->extra_elem[e] * m;
  uint8_t* tmp = (uint8_t*)malloc(need);
  if (!tmp) return ORC_OUT_OF_BOUNDS;
  gather3(c->data, idx, m, (float*)tmp);
  c->n = m;
  if (normals && c->normal) { gather3(c->normal, idx, m, (float*)tmp); c->n_normal = m; }
  if (colors && c->color) { gather3(c->color, idx, m, (float*)tmp); c->n_color = m; }
  if (intensity && c->intensity) { gather1(c->intensity, idx, m, (float*)tmp); c->n_intensity = m; }
  if (extra)
    for (int e = 0; e < ORC_MAX_EXTRA; ++e)
      if (c->extra[e]) { gatherb(c->extra[e], c->extra_elem[e], idx, m, tmp); c->n_extra[e] = m; }
  free(tmp);
  return ORC_OK;
}

static int check_index_fields(const orc_cloud* c, int normals, int colors,
                              int intensity, int extra) {
  if (normals && c->normal && c->n_normal < c->n) return ORC_OUT_OF_BOUNDS;
  if (colors && c->color && c->n_color < c->n) return ORC_OUT_OF_BOUNDS;
  if (intensity && c->intensity && c->n_intensity < c->n) return ORC_OUT_OF_BOUNDS;
  if (extra)
    for (int e = 0; e < ORC_MAX_EXTRA; ++e)
      if (c->extra[e] && c->n_extra[e] < c->n) return ORC_OUT_OF_BOUNDS;
  return ORC_OK;
}

static void rot(float* v, size_t n, float cs, float sn) { /* transforms.cpp:179-186 */
  for (size_t i = 0; i < n; ++i) {
    float px = v[3 * i], py = v[3 * i + 1];
    float a = px * cs, b = py * sn, x = a - b;
    float c = px * sn, d = py * cs, y = c + d;
    v[3 * i] = x;
    v[3 * i + 1] = y;
  }
}

/* FPS (App. C): start 0; d2 = (dx*dx + dy*dy) + dz*dz, no FMA; mind=min;
 * next = argmax mind, lowest index on ties, NaN never wins. */
static int op_fps(orc_cloud* c, int64_t m_in) {
  if (m_in <= 0) return ORC_OUT_OF_BOUNDS;
  size_t m = (size_t)m_in, n = c->n;
  if (n < m) return ORC_OUT_OF_BOUNDS;
  int st = check_index_fields(c, 1, 1, 1, 1);
  if (st) return st;
  float* mind = (float*)malloc(n * 4);
  size_t* idx = (size_t*)malloc(m * sizeof(size_t));
  for (size_t i = 0; i < n; ++i) mind[i] = INFINITY;
  size_t sel = 0;
  for (size_t k = 0; k < m; ++k) {
    idx[k] = sel;
    const float sx = c->data[3 * sel], sy = c->data[3 * sel + 1], sz = c->data[3 * sel + 2];
    size_t best = 0;
    float bestv = -INFINITY;
    int have = 0;
    for (size_t i = 0; i < n; ++i) {
      float dx = c->data[3 * i] - sx, dy = c->data[3 * i + 1] - sy, dz = c->data[3 * i + 2] - sz;
      float xx = dx * dx, yy = dy * dy, zz = dz * dz;
      float d = (xx + yy) + zz;
      if (d < mind[i]) mind[i] = d;
      if (!have || mind[i] > bestv) {
        if (mind[i] == mind[i]) { best = i; bestv = mind[i]; have = 1; }
      }
    }
    sel = best;
  }
  st = gather_all(c, idx, m, 1, 1, 1, 1);
  free(mind);
  free(idx);
  return st;
}

/* Voxel / grid subsample (App. C). */
typedef struct { uint64_t key; size_t i; } kv_t;
static int kv_cmp(const void* a, const void* b) {
  const kv_t* x = (const kv_t*)a;
  const kv_t* y = (const kv_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0); /* stable */
}

static int op_voxel(orc_cloud* c, const orc_params* p) {
  const size_t n = c->n;
  if (!(p->voxel_size > 0.0f)) return ORC_OUT_OF_BOUNDS;
  int st = check_index_fields(c, 1, 1, 1, 1);
  if (st) return st;
  float o[3];
  if (p->has_origin) {
    memcpy(o, p->origin, 12);
  } else {
    o[0] = c->data[0]; o[1] = c->data[1]; o[2] = c->data[2];
    for (size_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a)
        if (c->data[3 * i + a] < o[a]) o[a] = c->data[3 * i + a];
  }
  kv_t* kv = (kv_t*)malloc(n * sizeof(kv_t));
  for (size_t i = 0; i < n; ++i) {
    uint64_t key = 0;
    for (int a = 0; a < 3; ++a) {
      float d = c->data[3 * i + a] - o[a];
      float q = d / p->voxel_size;
      float f = floorf(q);
      if (!(f >= 0.0f && f < 2097152.0f)) { free(kv); return ORC_OUT_OF_BOUNDS; }
      key |= (uint64_t)(int32_t)f << (21 * a);
    }
    kv[i].key = key;
    kv[i].i = i;
  }
  qsort(kv, n, sizeof(kv_t), kv_cmp);
  /* segments */
  size_t v = 0;
  float* nd = (float*)malloc(12 * (n ? n : 1));
  float* nn = c->normal ? (float*)malloc(12 * (n ? n : 1)) : NULL;
  float* nc = c->color ? (float*)malloc(12 * (n ? n : 1)) : NULL;
  float* ni = c->intensity ? (float*)malloc(4 * (n ? n : 1)) : NULL;
  size_t* first = (size_t*)malloc(sizeof(size_t) * (n ? n : 1));
  for (size_t s = 0; s < n;) {
    size_t e = s;
    while (e < n && kv[e].key == kv[s].key) ++e;
    const double cnt = (double)(e - s);
    double sd[3] = {0, 0, 0}, sn[3] = {0, 0, 0}, sc[3] = {0, 0, 0}, si = 0;
    for (size_t k = s; k < e; ++k) {
      const size_t i = kv[k].i;
      for (int a = 0; a < 3; ++a) {
        sd[a] += (double)c->data[3 * i + a];
        if (nn) sn[a] += (double)c->normal[3 * i + a];
        if (nc) sc[a] += (double)c->color[3 * i + a];
      }
      if (ni) si += (double)c->intensity[i];
    }
    for (int a = 0; a < 3; ++a) {
      nd[3 * v + a] = (float)(sd[a] / cnt);
      if (nn) nn[3 * v + a] = (float)(sn[a] / cnt);
      if (nc) nc[3 * v + a] = (float)(sc[a] / cnt);
    }
    if (ni) ni[v] = (float)(si / cnt);
    if (c->counts) c->counts[v] = (int32_t)(e - s);
    first[v] = kv[s].i;
    ++v;
    s = e;
  }
  memcpy(c->data, nd, 12 * v);
  c->n = v;
  if (nn) { memcpy(c->normal, nn, 12 * v); c->n_normal = v; }
  if (nc) { memcpy(c->color, nc, 12 * v); c->n_color = v; }
  if (ni) { memcpy(c->intensity, ni, 4 * v); c->n_intensity = v; }
  if (c->counts) c->n_counts = v;
  /* extra per-point fields: value of the voxel's first point (original order) */
  uint8_t* tmp = (uint8_t*)malloc(16 * (v ? v : 1));
  for (int e = 0; e < ORC_MAX_EXTRA; ++e)
    if (c->extra[e]) { gatherb(c->extra[e], c->extra_elem[e], first, v, tmp); c->n_extra[e] = v; }
  free(tmp);
  free(first); free(nd); free(nn); free(nc); free(ni); free(kv);
  return ORC_OK;
}

static int op_range_crop(orc_cloud* c, const orc_params* p) {
  int st = check_index_fields(c, 1, 1, 1, 1);
  if (st) return st;
  size_t* idx = (size_t*)malloc(sizeof(size_t) * (c->n ? c->n : 1));
  size_t m = 0;
  for (size_t i = 0; i < c->n; ++i) {
    const float* q = c->data + 3 * i;
    if (q[0] >= p->lo[0] && q[0] <= p->hi[0] && q[1] >= p->lo[1] && q[1] <= p->hi[1] &&
        q[2] >= p->lo[2] && q[2] <= p->hi[2])
      idx[m++] = i;
  }
  st = gather_all(c, idx, m, 1, 1, 1, 1);
  free(idx);
  return st;
}

int orc_apply_map(int kind, const orc_params* p, orc_cloud* c, uint64_t seed) {
  /* get_points (transforms.cpp:33-41): "data" required and non-empty */
  if (!c->data) return ORC_MISSING_FIELD;
  if (c->n == 0) return ORC_EMPTY_CLOUD;
  orc_mt64 rng;
  orc_mt_seed(&rng, seed); /* transforms.cpp:114: constructed for every op */
  const size_t n = c->n;
  switch (kind) {
    case ORC_NORMALIZE: { /* transforms.cpp:122-147 */
      double cx = 0, cy = 0, cz = 0;
      for (size_t i = 0; i < n; ++i) {
        cx += c->data[3 * i];
        cy += c->data[3 * i + 1];
        cz += c->data[3 * i + 2];
      }
      const double dn = (double)n;
      cx /= dn; cy /= dn; cz /= dn;
      double s = 0;
      for (size_t i = 0; i < n; ++i) {
        double dx = c->data[3 * i] - cx, dy = c->data[3 * i + 1] - cy, dz = c->data[3 * i + 2] - cz;
        double xx = dx * dx, yy = dy * dy, zz = dz * dz;
        double r = sqrt((xx + yy) + zz);
        s = s < r ? r : s; /* std::max(s, r) */
      }
      for (size_t i = 0; i < n; ++i) {
        if (s == 0) {
          c->data[3 * i] = c->data[3 * i + 1] = c->data[3 * i + 2] = 0.0f;
        } else {
          c->data[3 * i] = (float)((c->data[3 * i] - cx) / s);
          c->data[3 * i + 1] = (float)((c->data[3 * i + 1] - cy) / s);
          c->data[3 * i + 2] = (float)((c->data[3 * i + 2] - cz) / s);
        }
      }
      return ORC_OK;
    }
    case ORC_TRANSLATE: { /* :149-157 */
      const float tx = orc_uniform_real(&rng, -0.2f, 0.2f);
      const float ty = orc_uniform_real(&rng, -0.2f, 0.2f);
      const float tz = orc_uniform_real(&rng, -0.2f, 0.2f);
      for (size_t i = 0; i < n; ++i) {
        c->data[3 * i] += tx;
        c->data[3 * i + 1] += ty;
        c->data[3 * i + 2] += tz;
      }
      return ORC_OK;
    }
    case ORC_JITTER: { /* :159-168 */
      orc_normal d = {0, 0.0f};
      for (size_t i = 0; i < 3 * n; ++i)
        c->data[i] += clampf_(orc_normal_draw(&d, &rng, 0.0f, 0.01f), -0.05f, 0.05f);
      return ORC_OK;
    }
    case ORC_ROTATE: { /* :169-190 */
      float theta = p && p->has_theta ? p->theta
                                      : orc_uniform_real(&rng, 0.0f, (float)(2.0 * M_PI));
      const float cs = cosf(theta), sn = sinf(theta);
      rot(c->data, n, cs, sn);
      if (c->normal && c->n_normal) rot(c->normal, c->n_normal, cs, sn);
      return ORC_OK;
    }
    case ORC_RANDOM_SCALE: { /* :191-200 */
      const float s = orc_uniform_real(&rng, 0.8f, 1.25f);
      for (size_t i = 0; i < 3 * n; ++i) c->data[i] *= s;
      return ORC_OK;
    }
    case ORC_FLIP_YZ: { /* :201-209 */
      if (orc_uniform_real(&rng, 0.0f, 1.0f) < 0.5f) {
        for (size_t i = 0; i < n; ++i) c->data[3 * i] = -c->data[3 * i];
        if (c->normal)
          for (size_t i = 0; i < c->n_normal; ++i) c->normal[3 * i] = -c->normal[3 * i];
      }
      return ORC_OK;
    }
    case ORC_COLOR_AUGMENT: { /* :210-219 */
      if (!c->color || c->n_color == 0) return ORC_MISSING_FIELD;
      for (size_t i = 0; i < 3 * c->n_color; ++i)
        c->color[i] = clampf_(c->color[i] + orc_uniform_real(&rng, -0.1f, 0.1f), 0.0f, 1.0f);
      return ORC_OK;
    }
    case ORC_RANDOM_CROP: { /* :220-271 */
      float lo[3] = {c->data[0], c->data[1], c->data[2]};
      float hi[3] = {c->data[0], c->data[1], c->data[2]};
      for (size_t i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
          const float v = c->data[3 * i + a];
          lo[a] = v < lo[a] ? v : lo[a]; /* std::min(lo, v) */
          hi[a] = hi[a] < v ? v : hi[a]; /* std::max(hi, v) */
        }
      float blo[3], bhi[3];
      for (int a = 0; a < 3; ++a) {
        const float extent = hi[a] - lo[a];
        const float f = orc_uniform_real(&rng, 0.7f, 1.0f);
        const float u = orc_uniform_real(&rng, 0.0f, 1.0f);
        const float t1 = u * extent;
        const float om = 1.0f - f;
        const float t2 = t1 * om;
        blo[a] = lo[a] + t2;
        const float ef = extent * f;
        bhi[a] = blo[a] + ef;
      }
      size_t* keep = (size_t*)malloc(sizeof(size_t) * n);
      size_t m = 0;
      for (size_t i = 0; i < n; ++i) {
        const float* q = c->data + 3 * i;
        if (q[0] >= blo[0] && q[0] <= bhi[0] && q[1] >= blo[1] && q[1] <= bhi[1] &&
            q[2] >= blo[2] && q[2] <= bhi[2])
          keep[m++] = i;
      }
      int st = ORC_OK;
      if (m > 0) {
        /* intensity only when it has at least as many entries as kept points */
        const int inten = c->intensity && c->n_intensity >= m;
        if (c->normal && c->n_normal < n) st = ORC_OUT_OF_BOUNDS;
        if (c->color && c->n_color < n) st = ORC_OUT_OF_BOUNDS;
        if (!st) {
          if (inten) { /* `if (i < in.size())` (:262) */
            size_t w = 0;
            float* t = (float*)malloc(4 * m);
            for (size_t k = 0; k < m; ++k)
              if (keep[k] < c->n_intensity) t[w++] = c->intensity[keep[k]];
            memcpy(c->intensity, t, 4 * w);
            c->n_intensity = w;
            free(t);
          }
          st = gather_all(c, keep, m, 1, 1, 0, 0);
        }
      }
      free(keep);
      return st;
    }
    case ORC_DOWNSAMPLE: { /* :272-299 */
      if (!p || p->num_points <= 0) return ORC_OUT_OF_BOUNDS;
      const size_t t = (size_t)p->num_points;
      if (t > c->cap) return ORC_OUT_OF_BOUNDS;
      int st = check_index_fields(c, 1, 1, p->gather_intensity, p->gather_extra);
      if (st) return st;
      size_t* idx = (size_t*)malloc(sizeof(size_t) * t);
      if (n >= t) {
        size_t* all = (size_t*)malloc(sizeof(size_t) * n);
        for (size_t i = 0; i < n; ++i) all[i] = i;
        for (size_t i = 0; i < t; ++i) {
          size_t j = (size_t)orc_uniform_int(&rng, i, n - 1);
          size_t tmp = all[i]; all[i] = all[j]; all[j] = tmp;
          idx[i] = all[i];
        }
        free(all);
      } else {
        for (size_t i = 0; i < t; ++i) idx[i] = (size_t)orc_uniform_int(&rng, 0, n - 1);
      }
      st = gather_all(c, idx, t, 1, 1, p->gather_intensity, p->gather_extra);
      free(idx);
      return st;
    }
    case ORC_FPS:
      return op_fps(c, p ? p->num_points : 0);
    case ORC_VOXEL:
      return op_voxel(c, p);
    case ORC_RANGE_CROP:
      return op_range_crop(c, p);
    default:
      return ORC_UNKNOWN_OP;
  }
}
