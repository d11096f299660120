// host_format.cpp — PcRecord header / index / page-head parsing and the
// dataset writer.  Behaviour follows the reference format code
// (proj/core/src/format.cpp, metadata.cpp, lz4_block.cpp); the byte layout
// is that of the reference so files written by either side interoperate
// (tests/test_format_host.py checks byte identity against the reference).
#include "host_format.h"

#include <cuda_runtime.h>

#include "kernels.h"
#include "page_encode.h"

#include <algorithm>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <thread>

#include "json.hpp"

namespace pcp {

using json = nlohmann::ordered_json;
namespace fs = std::filesystem;

const char* errc_name(int32_t st) {
  static const char* names[] = {
      "OK", "DuplicateField", "EmptySchema", "BadShape", "BadAlignment", "ColumnOutOfRange",
      "ChecksumMismatch", "CorruptPage", "SchemaMismatch", "IoFailure", "EmptyDataset",
      "BadMagic", "UnsupportedVersion", "CorruptHeader", "RangeOutOfBounds", "SchemaConflict",
      "OutOfRange", "NotPadded", "MalformedHeader", "TruncatedPayload", "UnsupportedProperty",
      "NoInputFiles", "ParseFailure", "Shutdown", "MissingField", "EmptyCloud", "UnknownOp",
      "OutOfBounds", "WorkerPanic", "ShapeMismatch", "StoreUnreachable", "MissingMetaIndex",
      "IntegrityFailure", "PipelineStopped", "InsufficientSamples", "SpaceExhausted",
      "UsageError"};
  if (st < 0 || st >= (int32_t)(sizeof(names) / sizeof(names[0]))) return "Unknown";
  return names[st];
}

// ---------------------------------------------------------------- schema
namespace {

const char* kind_name(int32_t k) {  // format.cpp:42-52
  switch (k) {
    case kBytes: return "bytes";
    case kInt32: return "int32";
    case kInt64: return "int64";
    case kFloat32: return "float32";
    case kFloat64: return "float64";
    case kString: return "string";
  }
  return "?";
}

int32_t kind_from(const std::string& n) {
  if (n == "bytes") return kBytes;
  if (n == "int32") return kInt32;
  if (n == "int64") return kInt64;
  if (n == "float32") return kFloat32;
  if (n == "float64") return kFloat64;
  if (n == "string") return kString;
  fail(kCorruptHeader, "unknown field type '" + n + "'");
}

json schema_json(const std::vector<FieldSpec>& s) {  // Schema::to_json (:69-79)
  json f = json::object();
  for (const auto& fs_ : s) {
    json ft;
    ft["type"] = kind_name(fs_.kind);
    if (!fs_.shape.empty()) ft["shape"] = fs_.shape;
    f[fs_.name] = ft;
  }
  return json{{"fields", f}};
}

std::vector<FieldSpec> schema_of(const json& j) {  // Schema::from_json (:81-92)
  std::vector<FieldSpec> s;
  if (!j.contains("fields") || !j["fields"].is_object())
    fail(kCorruptHeader, "schema missing fields");
  for (const auto& [name, ft] : j["fields"].items()) {
    FieldSpec f;
    f.name = name;
    f.kind = kind_from(ft.at("type").get<std::string>());
    if (ft.contains("shape")) f.shape = ft["shape"].get<std::vector<uint32_t>>();
    s.push_back(f);
  }
  return s;
}

void validate_schema(const std::vector<FieldSpec>& s) {  // :94-112
  if (s.empty()) fail(2, "schema has no fields");
  for (size_t i = 0; i < s.size(); ++i) {
    if (s[i].name.empty()) fail(3, "empty field name");
    for (char c : s[i].name)
      if ((unsigned char)c > 127) fail(3, "non-ASCII field name");
    for (size_t k = 0; k < i; ++k)
      if (s[k].name == s[i].name) fail(1, "field '" + s[i].name + "' declared twice");
    for (auto d : s[i].shape)
      if (d == 0) fail(3, "zero dimension in '" + s[i].name + "'");
    if (s[i].kind == kString && !s[i].shape.empty())
      fail(3, "string field '" + s[i].name + "' must be scalar");
  }
}

json header_json(const Header& h) {  // FileHeader::to_json (:313-332)
  json groups_j = json::array();
  for (const auto& g : h.groups)
    groups_j.push_back(json{{"group_id", g.group_id},
                            {"slice", g.slice},
                            {"first_sample", g.first_sample},
                            {"sample_count", g.sample_count},
                            {"scalar_page", {g.scalar_off, g.scalar_len}},
                            {"block_page", {g.block_off, g.block_len}},
                            {"blobs", g.blob_ranges},
                            {"blob_lens", g.blob_lens}});
  return json{{"version", h.version},
              {"total_size_bytes", h.total_size_bytes},
              {"scalar_page_size_bytes", h.scalar_page_size_bytes},
              {"block_page_size_bytes", h.block_page_size_bytes},
              {"schema", schema_json(h.schema)},
              {"slice_paths", h.slice_paths},
              {"group_index", groups_j}};
}

uint64_t header_byte_size(const Header& h) { return 4 + 2 + 4 + header_json(h).dump().size(); }

}  // namespace

std::vector<FieldSpec> schema_from_json(const std::string& text) {
  json j = json::parse(text, nullptr, false);
  if (j.is_discarded()) fail(kCorruptHeader, "schema is not valid JSON");
  auto s = schema_of(j);
  validate_schema(s);
  return s;
}

// ---------------------------------------------------------------- read
Header parse_header_json(const std::string& buf) {
  json j = json::parse(buf, nullptr, false);
  if (j.is_discarded()) fail(kCorruptHeader, "header is not valid JSON");
  Header h;
  try {  // FileHeader::from_json (:334-362)
    h.version = j.at("version").get<uint16_t>();
    h.total_size_bytes = j.at("total_size_bytes").get<uint64_t>();
    h.scalar_page_size_bytes = j.at("scalar_page_size_bytes").get<uint32_t>();
    h.block_page_size_bytes = j.at("block_page_size_bytes").get<uint32_t>();
    h.schema = schema_of(j.at("schema"));
    h.slice_paths = j.at("slice_paths").get<std::vector<std::string>>();
    for (const auto& gj : j.at("group_index")) {
      Group g;
      g.group_id = gj.at("group_id").get<uint32_t>();
      g.slice = gj.at("slice").get<uint32_t>();
      g.first_sample = gj.at("first_sample").get<uint64_t>();
      g.sample_count = gj.at("sample_count").get<uint32_t>();
      g.scalar_off = gj.at("scalar_page")[0].get<uint64_t>();
      g.scalar_len = gj.at("scalar_page")[1].get<uint64_t>();
      g.block_off = gj.at("block_page")[0].get<uint64_t>();
      g.block_len = gj.at("block_page")[1].get<uint64_t>();
      g.blob_ranges = gj.at("blobs").get<std::vector<std::array<uint64_t, 2>>>();
      g.blob_lens = gj.at("blob_lens").get<std::vector<std::vector<uint64_t>>>();
      h.groups.push_back(std::move(g));
    }
  } catch (const json::exception& e) {
    fail(kCorruptHeader, e.what());
  }
  // check_invariants (:364-376)
  if (h.slice_paths.empty()) fail(kCorruptHeader, "no slice paths");
  validate_schema(h.schema);
  for (const auto& g : h.groups) {
    if (g.slice >= h.slice_paths.size()) fail(kCorruptHeader, "group slice out of range");
    if (g.blob_ranges.size() != g.sample_count || g.blob_lens.size() != g.sample_count)
      fail(kCorruptHeader, "blob metadata count mismatch");
    for (const auto& r : g.blob_ranges)
      if (r[0] > r[1]) fail(kCorruptHeader, "blob range inverted");
  }
  h.header_bytes = header_byte_size(h);
  return h;
}

// FileHeader bytes (magic, version, JSON length, JSON) already in memory:
// parse + check_invariants (format.cpp:612-629,364-376); no slice-size checks.
Header parse_header_bytes(const uint8_t* p, size_t n) {
  if (n < 10) fail(kCorruptHeader, "file too short");
  if (std::memcmp(p, "PCRC", 4) != 0) fail(kBadMagic, "not a .pcrecord file");
  uint16_t version = 0;
  std::memcpy(&version, p + 4, 2);
  if (version != 1) fail(kUnsupportedVersion, "version " + std::to_string(version));
  uint32_t len = 0;
  std::memcpy(&len, p + 6, 4);
  if (10ull + len > n) fail(kCorruptHeader, "header truncated");
  return parse_header_json(std::string(reinterpret_cast<const char*>(p) + 10, len));
}

Header read_header(const std::string& primary) {
  std::ifstream f(primary, std::ios::binary);
  if (!f) fail(kIoFailure, "cannot open " + primary);
  char magic[4];
  if (!f.read(magic, 4)) fail(kCorruptHeader, "file too short");
  if (std::memcmp(magic, "PCRC", 4) != 0) fail(kBadMagic, "not a .pcrecord file");
  uint16_t version = 0;
  if (!f.read(reinterpret_cast<char*>(&version), 2)) fail(kCorruptHeader, "file too short");
  if (version != 1) fail(kUnsupportedVersion, "version " + std::to_string(version));
  uint32_t len = 0;
  if (!f.read(reinterpret_cast<char*>(&len), 4)) fail(kCorruptHeader, "file too short");
  std::string buf(len, '\0');
  if (!f.read(buf.data(), len)) fail(kCorruptHeader, "header truncated");
  Header h = parse_header_json(buf);
  // slice sizes (:630-652)
  const fs::path dir = fs::path(primary).parent_path();
  uint64_t on_disk = 0;
  std::vector<uint64_t> sizes;
  for (const auto& sp : h.slice_paths) {
    std::error_code ec;
    const auto sz = fs::file_size(dir / sp, ec);
    if (ec) fail(kCorruptHeader, "missing slice " + sp);
    sizes.push_back(sz);
    on_disk += sz;
  }
  if (on_disk != h.total_size_bytes) fail(kCorruptHeader, "total_size_bytes does not match disk");
  for (const auto& g : h.groups) {
    const uint64_t base = g.slice == 0 ? h.header_bytes : 0;
    if (base + g.block_off + g.block_len > sizes[g.slice] ||
        base + g.scalar_off + g.scalar_len > sizes[g.slice])
      fail(kCorruptHeader, "page range outside slice file");
  }
  return h;
}

std::vector<Entry> build_index(const Header& h) {
  std::vector<uint32_t> order(h.groups.size());
  for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    return h.groups[a].first_sample < h.groups[b].first_sample;
  });
  std::vector<Entry> out;
  for (uint32_t gi : order) {
    const Group& g = h.groups[gi];
    for (uint32_t r = 0; r < g.sample_count; ++r) {
      Entry e;
      e.shard_id = g.slice;
      e.group_id = g.group_id;
      e.group_index = gi;
      e.row = r;
      e.blob_start = g.blob_ranges[r][0];
      e.blob_end = g.blob_ranges[r][1];
      out.push_back(e);
    }
  }
  return out;
}

std::vector<uint8_t> read_slice_data(const Header& h, const std::string& dir, uint32_t slice) {
  const fs::path p = fs::path(dir) / h.slice_paths[slice];
  std::ifstream f(p, std::ios::binary);
  if (!f) fail(kIoFailure, "cannot open slice " + h.slice_paths[slice]);
  const uint64_t base = slice == 0 ? h.header_bytes : 0;
  const uint64_t sz = fs::file_size(p);
  if (sz < base) fail(kCorruptHeader, "slice shorter than its header");
  std::vector<uint8_t> buf(sz - base);
  f.seekg((std::streamoff)base);
  if (!buf.empty() && !f.read(reinterpret_cast<char*>(buf.data()), (std::streamsize)buf.size()))
    fail(kIoFailure, "short read of " + h.slice_paths[slice]);
  return buf;
}

PageHead parse_page_head(const uint8_t* p, uint64_t avail) {  // EncodedPage::deserialize
  if (avail < kPageHeaderBytes) fail(kCorruptPage, "record truncated");
  PageHead ph;
  ph.flags = p[0];
  std::memcpy(&ph.raw_len, p + 1, 8);
  std::memcpy(&ph.pay_len, p + 9, 8);
  std::memcpy(&ph.crc, p + 17, 4);
  if (kPageHeaderBytes + ph.pay_len > avail) fail(kCorruptPage, "page payload truncated");
  return ph;
}

// ---------------------------------------------------------------- codecs
uint32_t crc32_host(const uint8_t* p, size_t n) {
  static uint32_t tab[256];
  static bool ready = [] {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      tab[i] = c;
    }
    return true;
  }();
  (void)ready;
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = tab[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// Greedy single-probe LZ4 block matcher with the reference's parameters
// (lz4_block.cpp:11-17): 4-byte minimum match, 16-bit multiplicative hash,
// last 5 bytes literal, no match start in the last 12, offsets <= 65535.
std::vector<uint8_t> lz4_compress_host(const uint8_t* src, size_t n) {
  std::vector<uint8_t> out;
  out.reserve(n + n / 255 + 16);
  auto len_ext = [&](size_t v) {
    for (; v >= 255; v -= 255) out.push_back(255);
    out.push_back((uint8_t)v);
  };
  auto sequence = [&](size_t lit_from, size_t lit_to, size_t mlen, size_t dist) {
    const size_t lit = lit_to - lit_from;
    const size_t mcode = mlen ? mlen - 4 : 0;
    out.push_back((uint8_t)(((lit < 15 ? lit : 15) << 4) | (mlen ? (mcode < 15 ? mcode : 15) : 0)));
    if (lit >= 15) len_ext(lit - 15);
    out.insert(out.end(), src + lit_from, src + lit_to);
    if (mlen) {
      out.push_back((uint8_t)(dist & 0xff));
      out.push_back((uint8_t)(dist >> 8));
      if (mcode >= 15) len_ext(mcode - 15);
    }
  };
  if (n == 0) {
    out.push_back(0);
    return out;
  }
  size_t pos = 0, lit_start = 0;
  if (n > 12) {
    std::vector<uint32_t> last_seen(size_t(1) << 16, UINT32_MAX);
    auto word = [&](size_t i) {
      uint32_t v;
      std::memcpy(&v, src + i, 4);
      return v;
    };
    const size_t stop = n - 12, tail = n - 5;
    while (pos < stop) {
      const uint32_t w = word(pos);
      const uint32_t slot = (w * 2654435761u) >> 16;
      const uint32_t prev = last_seen[slot];
      last_seen[slot] = (uint32_t)pos;
      if (prev != UINT32_MAX && pos - prev <= 65535 && word(prev) == w) {
        size_t a = pos + 4, b = prev + 4;
        while (a < tail && src[a] == src[b]) ++a, ++b;
        sequence(lit_start, pos, a - pos, pos - prev);
        pos = lit_start = a;
      } else {
        ++pos;
      }
    }
  }
  sequence(lit_start, n, 0, 0);
  return out;
}

// ---------------------------------------------------------------- writer
namespace {

template <typename T>
void put(std::vector<uint8_t>& o, T v) {
  const auto* b = reinterpret_cast<const uint8_t*>(&v);
  o.insert(o.end(), b, b + sizeof(T));
}

struct EncodedGroup {
  Group g;
  std::vector<uint8_t> scalar, block;  // serialized pages
};

std::vector<uint8_t> finish_page(std::vector<uint8_t> post, uint64_t raw_len, uint8_t flags) {
  std::vector<uint8_t> lz = lz4_compress_host(post.data(), post.size());
  const bool use_lz = lz.size() < post.size();
  const std::vector<uint8_t>& pay = use_lz ? lz : post;
  std::vector<uint8_t> out;
  out.reserve(kPageHeaderBytes + pay.size());
  put<uint8_t>(out, flags | (use_lz ? kFlagOuterLz4 : kFlagStoredRaw));
  put<uint64_t>(out, raw_len);
  put<uint64_t>(out, pay.size());
  put<uint32_t>(out, crc32_host(pay.data(), pay.size()));
  out.insert(out.end(), pay.begin(), pay.end());
  return out;
}

// A group's raw pages and metadata (write_dataset :536-569) before encoding:
// the block page (blobs of every sample, bytes fields in schema order), its
// XOR-delta columns (delta_columns_for_group, :483-493) and the scalar page.
struct RawGroup {
  Group g;
  std::vector<uint8_t> block, scalar;
  std::vector<std::pair<uint64_t, uint64_t>> cols;  // (offset, length), width 4
};

RawGroup build_group(const std::vector<FieldSpec>& schema, const std::vector<SampleIn>& samples,
                     uint64_t first, uint32_t count) {
  RawGroup rg;
  Group& g = rg.g;
  g.first_sample = first;
  g.sample_count = count;
  std::vector<uint8_t>& block = rg.block;
  for (uint32_t r = 0; r < count; ++r) {
    const SampleIn& s = samples[first + r];
    const uint64_t start = block.size();
    std::vector<uint64_t> lens;
    for (size_t f = 0; f < schema.size(); ++f) {
      if (schema[f].kind != kBytes) continue;
      lens.push_back(s.values[f].size());
      block.insert(block.end(), s.values[f].begin(), s.values[f].end());
    }
    g.blob_ranges.push_back({start, block.size()});
    g.blob_lens.push_back(std::move(lens));
  }
  std::vector<uint8_t>& scalar = rg.scalar;  // append_scalar_record (:384-418)
  for (uint32_t r = 0; r < count; ++r) {
    const SampleIn& s = samples[first + r];
    put<uint64_t>(scalar, g.blob_ranges[r][0]);
    put<uint64_t>(scalar, g.blob_ranges[r][1]);
    put<uint32_t>(scalar, (uint32_t)g.blob_lens[r].size());
    for (auto l : g.blob_lens[r]) put<uint64_t>(scalar, l);
    for (size_t f = 0; f < schema.size(); ++f) {
      if (schema[f].kind == kBytes) continue;
      if (schema[f].kind == kString) put<uint32_t>(scalar, (uint32_t)s.values[f].size());
      scalar.insert(scalar.end(), s.values[f].begin(), s.values[f].end());
    }
  }
  for (uint32_t r = 0; r < count; ++r) {
    uint64_t at = g.blob_ranges[r][0];
    for (auto len : g.blob_lens[r]) {
      if (len >= 8 && len % 4 == 0) rg.cols.push_back({at, len});
      at += len;
    }
  }
  return rg;
}

EncodedGroup encode_group(const std::vector<FieldSpec>& schema,
                          const std::vector<SampleIn>& samples, uint64_t first, uint32_t count) {
  RawGroup rg = build_group(schema, samples, first, count);
  EncodedGroup eg;
  eg.g = std::move(rg.g);
  std::vector<uint8_t> work = rg.block;  // XOR-delta columns encoded in place
  for (const auto& [at, len] : rg.cols)
    for (uint64_t i = len; i >= 8; i -= 4) {
      uint32_t cur, prv;
      std::memcpy(&cur, rg.block.data() + at + i - 4, 4);
      std::memcpy(&prv, rg.block.data() + at + i - 8, 4);
      cur ^= prv;
      std::memcpy(work.data() + at + i - 4, &cur, 4);
    }
  eg.scalar = finish_page(rg.scalar, rg.scalar.size(), 0);
  eg.block = finish_page(std::move(work), rg.block.size(), rg.cols.empty() ? 0 : kFlagInnerDelta);
  return eg;
}

// The same pages encoded on the device (page_encode.cu), in batches of about
// 256 MB of raw pages: identical bytes.
std::vector<EncodedGroup> encode_groups_device(const std::vector<FieldSpec>& schema,
                                               const std::vector<SampleIn>& samples, uint32_t group_size,
                                               uint64_t num_groups, uint32_t n_threads, int device) {
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
    fail(kIoFailure, "no CUDA device: the device writer has no CPU fallback");
  if (device < 0 || device >= n_dev) fail(kOutOfBounds, "device index out of range");
  if (cudaSetDevice(device) != cudaSuccess) fail(kIoFailure, "cudaSetDevice failed");
  std::vector<RawGroup> raw(num_groups);
  {
    std::vector<std::thread> th;
    const uint32_t nt = std::max<uint32_t>(1, std::min<uint64_t>(n_threads, num_groups));
    for (uint32_t t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (uint64_t gi = t; gi < num_groups; gi += nt) {
          const uint64_t first = gi * group_size;
          raw[gi] = build_group(schema, samples, first,
                                (uint32_t)std::min<uint64_t>(group_size, samples.size() - first));
        }
      });
    for (auto& t : th) t.join();
  }
  std::vector<EncodedGroup> enc(num_groups);
  for (uint64_t gi = 0; gi < num_groups; ++gi) enc[gi].g = raw[gi].g;
  auto CKD = [](cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(kIoFailure, std::string("CUDA ") + what + ": " + cudaGetErrorString(e));
  };
  std::vector<uint32_t> shift(kShiftTabWords);
  build_shift_table(shift.data());
  uint32_t* d_shift = nullptr;
  CKD(cudaMalloc(&d_shift, shift.size() * 4), "malloc");
  CKD(cudaMemcpy(d_shift, shift.data(), shift.size() * 4, cudaMemcpyHostToDevice), "memcpy");
  // page list: scalar page then block page per group
  struct P {
    uint64_t g;
    bool block;
  };
  std::vector<P> all;
  for (uint64_t gi = 0; gi < num_groups; ++gi) all.push_back({gi, false}), all.push_back({gi, true});
  const uint64_t kBatch = 256ull << 20;
  size_t k = 0;
  while (k < all.size()) {
    size_t e = k;
    uint64_t bytes = 0;
    while (e < all.size()) {
      const auto& pg = all[e].block ? raw[all[e].g].block : raw[all[e].g].scalar;
      if (e > k && (bytes + pg.size() > kBatch || e - k >= 4096)) break;  // 256 KB hash table per page
      bytes += (pg.size() + 15) & ~uint64_t(15);
      ++e;
    }
    const uint32_t np = (uint32_t)(e - k);
    std::vector<EncPage> pages(np);
    std::vector<EncColumn> cols;
    std::vector<int> hb(np), he(np);
    uint64_t raw_at = 0, hash_at = 0, vis_at = 0, seq_at = 0, comp_at = 0;
    for (uint32_t i = 0; i < np; ++i) {
      const RawGroup& rg = raw[all[k + i].g];
      const auto& pg = all[k + i].block ? rg.block : rg.scalar;
      EncPage& p = pages[i];
      p.raw_off = raw_at;
      p.raw_len = pg.size();
      const uint64_t nh = pg.size() > 12 ? pg.size() - 12 : 0;
      p.hash_off = hash_at;
      hb[i] = (int)hash_at;
      he[i] = (int)(hash_at + nh);
      p.vis_off = vis_at;
      p.seq_off = seq_at;
      p.comp_off = comp_at;
      raw_at += (pg.size() + 15) & ~uint64_t(15);
      hash_at += nh;
      vis_at += nh / 32 + 2;
      seq_at += pg.size() / 4 + 2;
      comp_at += pg.size() + pg.size() / 255 + 64;
      if (all[k + i].block)
        for (const auto& [off, len] : rg.cols) cols.push_back({off, len, i, 0});
    }
    if (hash_at > (uint64_t)INT32_MAX) fail(kOutOfBounds, "page batch too large");
    const EncScratchSizes z = enc_scratch_sizes(raw_at, hash_at, np);
    std::vector<uint8_t> h_raw(raw_at + 16);
    for (uint32_t i = 0; i < np; ++i) {
      const auto& pg = all[k + i].block ? raw[all[k + i].g].block : raw[all[k + i].g].scalar;
      if (!pg.empty()) std::memcpy(h_raw.data() + pages[i].raw_off, pg.data(), pg.size());
    }
    // one device allocation carved into the buffers
    auto al = [](uint64_t v) { return (v + 255) & ~uint64_t(255); };
    uint64_t o = 0;
    const uint64_t o_raw = o; o += al(raw_at + 16);
    const uint64_t o_work = o; o += al(raw_at + 16);
    const uint64_t o_pages = o; o += al(sizeof(EncPage) * np);
    const uint64_t o_cols = o; o += al(sizeof(EncColumn) * cols.size() + 16);
    const uint64_t o_keys = o; o += al(z.keys + 16);
    const uint64_t o_keys2 = o; o += al(z.keys + 16);
    const uint64_t o_vals = o; o += al(z.vals + 16);
    const uint64_t o_vals2 = o; o += al(z.vals + 16);
    const uint64_t o_hb = o; o += al(4ull * np);
    const uint64_t o_he = o; o += al(4ull * np);
    const uint64_t o_prev = o; o += al(z.prev + 16);
    const uint64_t o_vis = o; o += al(z.visited + 16);
    const uint64_t o_seqs = o; o += al(sizeof(EncSeq) * seq_at + 16);
    const uint64_t o_nseq = o; o += al(4ull * np);
    const uint64_t o_comp = o; o += al(comp_at + 16);
    const uint64_t o_clen = o; o += al(8ull * np);
    const uint64_t o_crc = o; o += al(4ull * np);
    const uint64_t o_cub = o; o += al(z.cub);
    uint8_t* d = nullptr;
    CKD(cudaMalloc(&d, o), "malloc");
    EncArgs a{};
    a.n_pages = np;
    a.n_cols = (uint32_t)cols.size();
    a.raw_total = raw_at;
    a.hash_total = hash_at;
    a.raw = d + o_raw;
    a.work = d + o_work;
    a.pages = reinterpret_cast<const EncPage*>(d + o_pages);
    a.cols = reinterpret_cast<const EncColumn*>(d + o_cols);
    a.keys = reinterpret_cast<uint32_t*>(d + o_keys);
    a.keys_alt = reinterpret_cast<uint32_t*>(d + o_keys2);
    a.vals = reinterpret_cast<uint32_t*>(d + o_vals);
    a.vals_alt = reinterpret_cast<uint32_t*>(d + o_vals2);
    a.hash_begin = reinterpret_cast<const int*>(d + o_hb);
    a.hash_end = reinterpret_cast<const int*>(d + o_he);
    a.prev = reinterpret_cast<uint32_t*>(d + o_prev);
    a.visited = reinterpret_cast<uint32_t*>(d + o_vis);
    a.visited_bytes = z.visited;
    a.seqs = reinterpret_cast<EncSeq*>(d + o_seqs);
    a.n_seqs = reinterpret_cast<uint32_t*>(d + o_nseq);
    a.comp = d + o_comp;
    a.comp_len = reinterpret_cast<uint64_t*>(d + o_clen);
    a.crc = reinterpret_cast<uint32_t*>(d + o_crc);
    a.shift_tab = d_shift;
    a.cub = d + o_cub;
    a.cub_bytes = z.cub;
    CKD(cudaMemcpy(d + o_raw, h_raw.data(), raw_at, cudaMemcpyHostToDevice), "memcpy");
    CKD(cudaMemcpy(d + o_pages, pages.data(), sizeof(EncPage) * np, cudaMemcpyHostToDevice), "memcpy");
    if (!cols.empty())
      CKD(cudaMemcpy(d + o_cols, cols.data(), sizeof(EncColumn) * cols.size(), cudaMemcpyHostToDevice), "memcpy");
    CKD(cudaMemcpy(d + o_hb, hb.data(), 4ull * np, cudaMemcpyHostToDevice), "memcpy");
    CKD(cudaMemcpy(d + o_he, he.data(), 4ull * np, cudaMemcpyHostToDevice), "memcpy");
    CKD(launch_encode_pages(a, nullptr), "page encode");
    CKD(cudaDeviceSynchronize(), "page encode");
    std::vector<uint64_t> clen(np);
    std::vector<uint32_t> crc(np);
    CKD(cudaMemcpy(clen.data(), d + o_clen, 8ull * np, cudaMemcpyDeviceToHost), "memcpy");
    CKD(cudaMemcpy(crc.data(), d + o_crc, 4ull * np, cudaMemcpyDeviceToHost), "memcpy");
    for (uint32_t i = 0; i < np; ++i) {
      const P& pp = all[k + i];
      const RawGroup& rg = raw[pp.g];
      const bool lz = clen[i] < pages[i].raw_len;  // finish_page: LZ4 only when it shrinks
      const uint64_t pay = lz ? clen[i] : pages[i].raw_len;
      std::vector<uint8_t> out(kPageHeaderBytes + pay);
      const uint8_t flags = (pp.block && !rg.cols.empty() ? kFlagInnerDelta : 0) | (lz ? kFlagOuterLz4 : kFlagStoredRaw);
      out[0] = flags;
      std::memcpy(out.data() + 1, &pages[i].raw_len, 8);
      std::memcpy(out.data() + 9, &pay, 8);
      std::memcpy(out.data() + 17, &crc[i], 4);
      if (pay)
        CKD(cudaMemcpy(out.data() + kPageHeaderBytes, d + (lz ? o_comp + pages[i].comp_off : o_work + pages[i].raw_off),
                       pay, cudaMemcpyDeviceToHost), "memcpy");
      (pp.block ? enc[pp.g].block : enc[pp.g].scalar) = std::move(out);
    }
    cudaFree(d);
    k = e;
  }
  cudaFree(d_shift);
  return enc;
}

}  // namespace

Header write_dataset(const std::vector<FieldSpec>& schema, const std::vector<SampleIn>& samples,
                     uint32_t slice_count, uint32_t group_size, const std::string& out_dir,
                     const std::string& stem, uint32_t n_threads, int device) {
  validate_schema(schema);
  if (samples.empty()) fail(kEmptyDataset, "no samples to write");
  if (slice_count < 1 || group_size < 1) fail(kOutOfBounds, "slice_count and group_size must be >= 1");
  for (const auto& s : samples) {  // validate_sample (:125-159)
    if (s.values.size() != schema.size()) fail(kSchemaMismatch, "field count mismatch");
    for (size_t f = 0; f < schema.size(); ++f) {
      const auto& fs_ = schema[f];
      const uint64_t n = fs_.elems();
      const uint64_t nb = s.values[f].size();
      uint64_t es = 0;
      switch (fs_.kind) {
        case kBytes:
          if (!fs_.shape.empty() && nb % n) fail(kSchemaMismatch, "blob length of '" + fs_.name + "' not divisible by shape");
          break;
        case kInt32: case kFloat32: es = 4; break;
        case kInt64: case kFloat64: es = 8; break;
        default: break;
      }
      if (es && nb != es * n) fail(kSchemaMismatch, "element count mismatch for '" + fs_.name + "'");
    }
  }
  const uint64_t num_groups = (samples.size() + group_size - 1) / group_size;
  const uint64_t groups_per_slice = (num_groups + slice_count - 1) / slice_count;
  std::vector<EncodedGroup> enc;
  if (device >= 0) {
    enc = encode_groups_device(schema, samples, group_size, num_groups, n_threads, device);
  } else {
    enc.resize(num_groups);
    n_threads = std::max<uint32_t>(1, std::min<uint64_t>(n_threads, num_groups));
    std::vector<std::thread> th;
    for (uint32_t t = 0; t < n_threads; ++t)
      th.emplace_back([&, t] {
        for (uint64_t gi = t; gi < num_groups; gi += n_threads) {
          const uint64_t first = gi * group_size;
          const uint32_t cnt = (uint32_t)std::min<uint64_t>(group_size, samples.size() - first);
          enc[gi] = encode_group(schema, samples, first, cnt);
        }
      });
    for (auto& t : th) t.join();
  }

  Header h;
  h.schema = schema;
  h.slice_paths.resize(slice_count);
  for (uint32_t s = 0; s < slice_count; ++s)
    h.slice_paths[s] = s == 0 ? stem + ".pcrecord" : stem + ".pcrecord" + std::to_string(s);
  std::vector<uint64_t> slice_size(slice_count, 0);
  std::vector<uint32_t> per_slice(slice_count, 0);
  for (uint64_t gi = 0; gi < num_groups; ++gi) {
    Group& g = enc[gi].g;
    g.slice = (uint32_t)std::min<uint64_t>(gi / groups_per_slice, slice_count - 1);
    g.group_id = per_slice[g.slice]++;
    g.scalar_off = slice_size[g.slice];
    g.scalar_len = enc[gi].scalar.size();
    g.block_off = g.scalar_off + g.scalar_len;
    g.block_len = enc[gi].block.size();
    slice_size[g.slice] = g.block_off + g.block_len;
    h.scalar_page_size_bytes = std::max<uint32_t>(h.scalar_page_size_bytes, (uint32_t)g.scalar_len);
    h.block_page_size_bytes = std::max<uint32_t>(h.block_page_size_bytes, (uint32_t)g.block_len);
    h.groups.push_back(g);
  }
  uint64_t data_total = 0;
  for (auto v : slice_size) data_total += v;
  h.total_size_bytes = 0;
  for (int i = 0; i < 10; ++i) {  // :583-590
    const uint64_t total = header_byte_size(h) + data_total;
    if (total == h.total_size_bytes) break;
    h.total_size_bytes = total;
  }
  fs::create_directories(out_dir);
  for (uint32_t s = 0; s < slice_count; ++s) {
    std::ofstream f(fs::path(out_dir) / h.slice_paths[s], std::ios::binary);
    if (!f) fail(kIoFailure, "cannot open " + h.slice_paths[s]);
    if (s == 0) {
      const std::string j = header_json(h).dump();
      const uint16_t ver = h.version;
      const uint32_t len = (uint32_t)j.size();
      f.write("PCRC", 4);
      f.write(reinterpret_cast<const char*>(&ver), 2);
      f.write(reinterpret_cast<const char*>(&len), 4);
      f.write(j.data(), (std::streamsize)j.size());
    }
    for (uint64_t gi = 0; gi < num_groups; ++gi) {
      if (h.groups[gi].slice != s) continue;
      f.write(reinterpret_cast<const char*>(enc[gi].scalar.data()), (std::streamsize)enc[gi].scalar.size());
      f.write(reinterpret_cast<const char*>(enc[gi].block.data()), (std::streamsize)enc[gi].block.size());
    }
    if (!f) fail(kIoFailure, "short write to " + h.slice_paths[s]);
  }
  h.header_bytes = header_byte_size(h);
  return h;
}

}  // namespace pcp
