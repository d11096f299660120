// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle).
//
// A thin extern "C" layer over the *unmodified* reference library
// (/root/reference/proj/core/src/*.cpp, compiled in place by oracle/Makefile
// into oracle/_ref/libpcpipe_ref.so).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.  Nothing on
// the product path links or calls this file.
//
// Every function forwards to the reference symbol named in its comment, so the
// outputs are the reference's own.  Samples/batches cross this ABI in a tiny
// TLV format (see tlv_* below) that tests/oracle_ffi.py parses.
//
//   sample  := u32 n_fields { u16 name_len, name, u8 kind, u64 nbytes, bytes }
//   kind    := 0 bytes | 1 int32 | 2 int64 | 3 float32 | 4 float64 | 5 string
//   batches := u32 n_batches { u64 epoch, u64 batch_index, u32 n_samples, sample* }

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <map>
#include <vector>

#include "pcpipe/bench.hpp"
#include "pcpipe/distributed.hpp"
#include "pcpipe/errors.hpp"
#include "pcpipe/format.hpp"
#include "pcpipe/lz4_block.hpp"
#include "pcpipe/metadata.hpp"
#include "pcpipe/pipeline.hpp"
#include "pcpipe/transforms.hpp"
#include "pcpipe_oracle.h"

using namespace pcpipe;

namespace {

thread_local std::string g_err;
thread_local int g_errc = 0;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_errc = 0;
    g_err.clear();
    return 0;
  } catch (const PcError& e) {
    g_errc = static_cast<int>(e.code()) + 1;
    g_err = e.what();
    return g_errc;
  } catch (const std::exception& e) {
    g_errc = 1000;
    g_err = e.what();
    return g_errc;
  }
}

struct Reader {
  const std::uint8_t* p;
  std::size_t n;
  std::size_t pos = 0;
  template <typename T>
  T get() {
    if (pos + sizeof(T) > n) throw std::runtime_error("tlv truncated");
    T v;
    std::memcpy(&v, p + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  const std::uint8_t* take(std::size_t k) {
    if (pos + k > n) throw std::runtime_error("tlv truncated");
    const auto* r = p + pos;
    pos += k;
    return r;
  }
};

template <typename T>
void put(std::vector<std::uint8_t>& out, T v) {
  const auto* b = reinterpret_cast<const std::uint8_t*>(&v);
  out.insert(out.end(), b, b + sizeof(T));
}

template <typename T>
std::vector<T> vec_of(const std::uint8_t* b, std::size_t nbytes) {
  std::vector<T> v(nbytes / sizeof(T));
  std::memcpy(v.data(), b, v.size() * sizeof(T));
  return v;
}

Sample read_sample_tlv(Reader& r) {
  Sample s;
  const auto nf = r.get<std::uint32_t>();
  for (std::uint32_t f = 0; f < nf; ++f) {
    const auto nl = r.get<std::uint16_t>();
    std::string name(reinterpret_cast<const char*>(r.take(nl)), nl);
    const auto kind = r.get<std::uint8_t>();
    const auto nb = r.get<std::uint64_t>();
    const auto* b = r.take(nb);
    switch (kind) {
      case 0: s.values[name] = Blob(b, b + nb); break;
      case 1: s.values[name] = vec_of<std::int32_t>(b, nb); break;
      case 2: s.values[name] = vec_of<std::int64_t>(b, nb); break;
      case 3: s.values[name] = vec_of<float>(b, nb); break;
      case 4: s.values[name] = vec_of<double>(b, nb); break;
      default: s.values[name] = std::string(reinterpret_cast<const char*>(b), nb); break;
    }
  }
  return s;
}

void write_sample_tlv(std::vector<std::uint8_t>& out, const Sample& s) {
  put<std::uint32_t>(out, static_cast<std::uint32_t>(s.values.size()));
  for (const auto& [name, v] : s.values) {
    put<std::uint16_t>(out, static_cast<std::uint16_t>(name.size()));
    out.insert(out.end(), name.begin(), name.end());
    put<std::uint8_t>(out, static_cast<std::uint8_t>(v.index()));
    std::visit(
        [&](const auto& x) {
          using T = std::decay_t<decltype(x)>;
          std::size_t nb;
          const std::uint8_t* b;
          if constexpr (std::is_same_v<T, std::string>) {
            nb = x.size();
            b = reinterpret_cast<const std::uint8_t*>(x.data());
          } else {
            nb = x.size() * sizeof(typename T::value_type);
            b = reinterpret_cast<const std::uint8_t*>(x.data());
          }
          put<std::uint64_t>(out, nb);
          out.insert(out.end(), b, b + nb);
        },
        v);
  }
}

void hand_out(const std::vector<std::uint8_t>& v, std::uint8_t** out,
              std::size_t* out_len) {
  *out_len = v.size();
  *out = static_cast<std::uint8_t*>(std::malloc(v.empty() ? 1 : v.size()));
  if (!v.empty()) std::memcpy(*out, v.data(), v.size());
}

std::vector<ColumnRange> cols_of(const std::uint64_t* off, const std::uint64_t* len,
                                 std::size_t n) {
  std::vector<ColumnRange> c(n);
  for (std::size_t i = 0; i < n; ++i) c[i] = {off[i], len[i], 4};
  return c;
}

}  // namespace

extern "C" {

int ref_last_errc(void) { return g_errc; }
const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// format.cpp:163-166
std::uint32_t ref_crc32(const std::uint8_t* b, std::size_t n) {
  return crc32_of(std::span<const std::uint8_t>(b, n));
}

// transforms.cpp:82-96
std::uint64_t ref_mix_seed(std::uint64_t base, std::uint64_t epoch,
                           std::uint64_t index, std::uint64_t op) {
  return mix_seed(base, epoch, index, op);
}

// lz4_block.cpp:33-110
std::size_t ref_lz4_compress(const std::uint8_t* src, std::size_t n,
                             std::uint8_t* dst, std::size_t cap) {
  return lz4::compress(src, n, dst, cap);
}

// lz4_block.cpp:113-156
int ref_lz4_decompress(const std::uint8_t* src, std::size_t n, std::uint8_t* dst,
                       std::size_t raw_len) {
  return guarded([&] { lz4::decompress(src, n, dst, raw_len); });
}

// format.cpp:168-195
int ref_xor_delta(int encode, const std::uint8_t* in, std::size_t n,
                  std::uint32_t width, std::uint8_t** out, std::size_t* out_len) {
  return guarded([&] {
    auto sp = std::span<const std::uint8_t>(in, n);
    hand_out(encode ? xor_delta_encode(sp, width) : xor_delta_decode(sp, width),
             out, out_len);
  });
}

// format.cpp:198-241 + EncodedPage::serialize_to (:281-287)
int ref_encode_block_page(const std::uint8_t* raw, std::size_t n,
                          const std::uint64_t* col_off, const std::uint64_t* col_len,
                          std::size_t ncols, int scalar, std::uint8_t** out,
                          std::size_t* out_len) {
  return guarded([&] {
    auto sp = std::span<const std::uint8_t>(raw, n);
    auto cols = cols_of(col_off, col_len, ncols);
    EncodedPage p = scalar ? encode_scalar_page(sp) : encode_block_page(sp, cols);
    Blob b;
    p.serialize_to(b);
    hand_out(b, out, out_len);
  });
}

// EncodedPage::deserialize (format.cpp:289-299) + decode_block_page (:243-266)
int ref_decode_block_page(const std::uint8_t* page, std::size_t n,
                          const std::uint64_t* col_off, const std::uint64_t* col_len,
                          std::size_t ncols, std::uint8_t** out, std::size_t* out_len) {
  return guarded([&] {
    auto p = EncodedPage::deserialize(std::span<const std::uint8_t>(page, n));
    auto cols = cols_of(col_off, col_len, ncols);
    hand_out(decode_block_page(p, cols), out, out_len);
  });
}

// transforms.cpp:98-306
int ref_apply_map(const char* kind, const char* params_json,
                  const std::uint8_t* sample, std::size_t n, std::uint64_t seed,
                  std::uint8_t** out, std::size_t* out_len) {
  return guarded([&] {
    Reader r{sample, n};
    Sample s = read_sample_tlv(r);
    json params = (params_json && *params_json) ? json::parse(params_json)
                                                : json::object();
    Sample o = apply_map(map_kind_from_name(kind), params, std::move(s), seed);
    std::vector<std::uint8_t> buf;
    write_sample_tlv(buf, o);
    hand_out(buf, out, out_len);
  });
}

// format.cpp:499-610
int ref_write_dataset(const char* out_dir, const char* stem, const char* schema_json,
                      const std::uint8_t* samples, std::size_t n,
                      std::uint32_t n_samples, std::uint32_t slice_count,
                      std::uint32_t group_size) {
  return guarded([&] {
    Schema schema = Schema::from_json(json::parse(schema_json));
    Reader r{samples, n};
    std::vector<Sample> v;
    v.reserve(n_samples);
    for (std::uint32_t i = 0; i < n_samples; ++i) v.push_back(read_sample_tlv(r));
    WriteOptions o;
    o.slice_count = slice_count;
    o.group_size = group_size;
    o.stem = stem;
    write_dataset(v, schema, o, out_dir);
  });
}

// DatasetReader::read_sample over build_index (format.cpp:729-757,
// metadata.cpp:20-52); entry ids index the (optionally padded+sharded) table.
int ref_read_samples(const char* primary, const std::uint64_t* ids, std::size_t n_ids,
                     std::uint8_t** out, std::size_t* out_len) {
  return guarded([&] {
    DatasetReader rd(primary);
    IndexTable idx = build_index({rd.header()});
    std::vector<std::uint8_t> buf;
    put<std::uint32_t>(buf, static_cast<std::uint32_t>(n_ids));
    for (std::size_t i = 0; i < n_ids; ++i)
      write_sample_tlv(buf, rd.read_sample(locate(idx, ids[i])));
    hand_out(buf, out, out_len);
  });
}

// Index JSON (metadata.cpp:8-18) after optional pad_for_shards (:60-74) and
// shard_index (distributed.cpp:13-27).
int ref_index_json(const char* primary, std::uint32_t num_shards, std::uint32_t shard_id,
                   std::uint8_t** out, std::size_t* out_len) {
  return guarded([&] {
    DatasetReader rd(primary);
    IndexTable idx = build_index({rd.header()});
    if (num_shards > 0) {
      idx = pad_for_shards(idx, num_shards);
      idx = shard_index(idx, ShardSpec{num_shards, shard_id});
    }
    const std::string s = idx.to_json().dump();
    hand_out(std::vector<std::uint8_t>(s.begin(), s.end()), out, out_len);
  });
}

namespace {
IndexTable select_entries(const IndexTable& full, const std::uint64_t* ids,
                          std::size_t n_ids) {
  if (!ids) return full;
  IndexTable t;
  t.total_real_samples = full.total_real_samples;
  for (std::size_t i = 0; i < n_ids; ++i) {
    const auto& e = locate(full, ids[i]);
    t.task_list.push_back(e.task);
    t.sample_meta_list.push_back(e);
  }
  return t;
}
}  // namespace

// Pipeline over dataset_source (pcpipe_main.cpp:49-53) → every batch, every
// sample (un-stacked so ragged ops can be compared too). ids (optional) is the
// entry list the source walks, e.g. one GPU's shard.
int ref_run_pipeline(const char* primary, const char* graph_json,
                     const std::uint64_t* ids, std::size_t n_ids, std::uint64_t epochs,
                     std::uint8_t** out, std::size_t* out_len) {
  return guarded([&] {
    auto rd = std::make_shared<DatasetReader>(primary);
    auto idx = std::make_shared<IndexTable>(
        select_entries(build_index({rd->header()}), ids, n_ids));
    PipelineGraph g = PipelineGraph::from_json(json::parse(graph_json));
    PipelineOptions opts;
    opts.epochs = epochs;
    Pipeline p(g,
               [rd, idx](std::uint64_t, std::uint64_t i) {
                 return rd->read_sample(idx->sample_meta_list[i]);
               },
               idx->size(), opts);
    p.start();
    std::vector<std::uint8_t> buf;
    std::vector<Batch> batches;
    while (auto b = p.next_batch()) batches.push_back(std::move(*b));
    p.stop();
    put<std::uint32_t>(buf, static_cast<std::uint32_t>(batches.size()));
    for (const auto& b : batches) {
      put<std::uint64_t>(buf, b.epoch);
      put<std::uint64_t>(buf, b.batch_index);
      put<std::uint32_t>(buf, static_cast<std::uint32_t>(b.samples.size()));
      for (const auto& s : b.samples) write_sample_tlv(buf, s);
    }
    hand_out(buf, out, out_len);
  });
}

// run_benchmark (bench.cpp:43-96): warm-up batch excluded, mean over repeats.
// Graph workers are whatever the graph JSON says.
int ref_bench_pipeline(const char* primary, const char* graph_json,
                       std::uint32_t repeats, const std::uint64_t* ids,
                       std::size_t n_ids, double* cost_time_s, std::uint64_t* items,
                       std::uint64_t* batches, double* avg_cpu_percent) {
  return guarded([&] {
    auto rd = std::make_shared<DatasetReader>(primary);
    auto idx = std::make_shared<IndexTable>(
        select_entries(build_index({rd->header()}), ids, n_ids));
    PipelineGraph g = PipelineGraph::from_json(json::parse(graph_json));
    SourceFn src = [rd, idx](std::uint64_t, std::uint64_t i) {
      return rd->read_sample(idx->sample_meta_list[i]);
    };
    BenchReport rep = run_benchmark(g, src, idx->size(), repeats, 50);
    *cost_time_s = rep.cost_time_s;
    *items = rep.items;
    *batches = rep.batches;
    *avg_cpu_percent = rep.avg_cpu_percent;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// CPU baseline for chains with App. C ops (fps / voxel / grid_subsample /
// range_crop and the "gather" extension), which the reference lacks.  The
// reference Pipeline runs as shipped; its SourceFn (pipeline.cpp:442-462,
// source workers = all host threads) reads the sample with the reference
// reader and applies the chain's prefix up to the last non-reference step:
// reference ops through the reference apply_map, App. C ops through the C
// restatement (pcpipe_oracle.c, compiled into this library), each seeded with
// the reference mix_seed(base, epoch, index, op_id).  The remaining
// reference-op suffix runs in the Pipeline's own map workers.
namespace {

struct Step {
  std::string map;
  json params;
  std::uint64_t op_id;
};

bool is_ref_op(const Step& st) {
  static const char* k[] = {"normalize", "translate", "jitter", "rotate", "random_scale",
                            "flip_yz", "color_augment", "random_crop", "downsample"};
  if (st.params.is_object() && st.params.contains("gather")) return false;
  for (const char* n : k)
    if (st.map == n) return true;
  return false;
}

Blob& blob_of(Sample& s, const std::string& name) { return std::get<Blob>(s.values.at(name)); }
bool has_blob(const Sample& s, const std::string& name) {
  auto it = s.values.find(name);
  return it != s.values.end() && std::holds_alternative<Blob>(it->second);
}

// Orc.apply_map (oracle/ffi.py) in C++: Sample <-> orc_cloud.
Sample orc_apply(const Step& st, Sample s, std::uint64_t seed) {
  static const std::map<std::string, int> kinds = {
      {"normalize", ORC_NORMALIZE}, {"translate", ORC_TRANSLATE}, {"jitter", ORC_JITTER},
      {"rotate", ORC_ROTATE}, {"random_scale", ORC_RANDOM_SCALE}, {"flip_yz", ORC_FLIP_YZ},
      {"color_augment", ORC_COLOR_AUGMENT}, {"random_crop", ORC_RANDOM_CROP},
      {"downsample", ORC_DOWNSAMPLE}, {"fps", ORC_FPS}, {"voxel", ORC_VOXEL},
      {"grid_subsample", ORC_VOXEL}, {"range_crop", ORC_RANGE_CROP}};
  const auto kit = kinds.find(st.map);
  if (kit == kinds.end()) fail(Errc::kUnknownOp, "unknown map '" + st.map + "'");
  const json p = st.params.is_object() ? st.params : json::object();
  std::vector<std::string> gather;
  if (p.contains("gather"))
    for (const auto& g : p["gather"]) gather.push_back(g.get<std::string>());
  if (!has_blob(s, "data")) fail(Errc::kMissingField, "sample has no 'data' coordinates");
  const char* p3[3] = {"data", "normal", "color"};
  bool present[3] = {false, false, false};
  std::size_t len3[3] = {0, 0, 0};
  for (int k = 0; k < 3; ++k) {
    if (!has_blob(s, p3[k])) continue;
    const Blob& b = blob_of(s, p3[k]);
    if (k > 0 && b.empty()) continue;
    if (b.size() % 12) fail(Errc::kMissingField, std::string(p3[k]) + " is not an Nx3 float32 blob");
    present[k] = true;
    len3[k] = b.size() / 12;
  }
  const std::size_t n = len3[0];
  if (n == 0) fail(Errc::kEmptyCloud, "zero points");
  const std::int64_t tgt = p.value("num_points", std::int64_t{0});
  std::size_t cap = std::max<std::size_t>({n, (std::size_t)std::max<std::int64_t>(tgt, 0), len3[1], len3[2], 1});
  std::vector<float> buf3[3];
  orc_cloud cl{};
  float** dst3[3] = {&cl.data, &cl.normal, &cl.color};
  for (int k = 0; k < 3; ++k) {
    if (!present[k]) continue;
    buf3[k].assign(cap * 3, 0.0f);
    const Blob& b = blob_of(s, p3[k]);
    std::memcpy(buf3[k].data(), b.data(), b.size());
    *dst3[k] = buf3[k].data();
  }
  cl.n = n;
  cl.n_normal = present[1] ? len3[1] : 0;
  cl.n_color = present[2] ? len3[2] : 0;
  std::vector<float> bi;
  if (has_blob(s, "intensity") && !blob_of(s, "intensity").empty()) {
    const Blob& b = blob_of(s, "intensity");
    const std::size_t ni = b.size() / 4;
    bi.assign(std::max(cap, ni), 0.0f);
    std::memcpy(bi.data(), b.data(), ni * 4);
    cl.intensity = bi.data();
    cl.n_intensity = ni;
  }
  std::vector<std::string> extra;
  for (const auto& g : gather)
    if (g != "intensity" && s.values.count(g)) extra.push_back(g);
  if (extra.size() > ORC_MAX_EXTRA) extra.resize(ORC_MAX_EXTRA);
  std::vector<std::vector<std::uint8_t>> eb(extra.size());
  for (std::size_t e = 0; e < extra.size(); ++e) {
    const Blob& b = blob_of(s, extra[e]);
    const std::size_t es = std::max<std::size_t>(1, b.size() / n);
    eb[e].assign(cap * es, 0);
    std::memcpy(eb[e].data(), b.data(), std::min(b.size(), eb[e].size()));
    cl.extra[e] = eb[e].data();
    cl.extra_elem[e] = es;
    cl.n_extra[e] = b.size() / es;
  }
  std::vector<std::int32_t> counts;
  const bool want_counts = (st.map == "voxel" || st.map == "grid_subsample") &&
                           p.value("counts", st.map == "voxel");
  if (want_counts) {
    counts.assign(cap, 0);
    cl.counts = counts.data();
  }
  cl.cap = cap;
  orc_params op{};
  if (p.contains("theta")) {
    op.has_theta = 1;
    op.theta = p["theta"].get<float>();
  }
  op.num_points = tgt;
  op.gather_intensity = std::find(gather.begin(), gather.end(), "intensity") != gather.end();
  op.gather_extra = !extra.empty();
  op.voxel_size = p.value("voxel_size", 0.0f);
  if (p.contains("origin")) {
    op.has_origin = 1;
    for (int k = 0; k < 3; ++k) op.origin[k] = p["origin"][k].get<float>();
  }
  if (p.contains("lo"))
    for (int k = 0; k < 3; ++k) op.lo[k] = p["lo"][k].get<float>();
  if (p.contains("hi"))
    for (int k = 0; k < 3; ++k) op.hi[k] = p["hi"][k].get<float>();
  const int st_code = orc_apply_map(kit->second, &op, &cl, seed);
  if (st_code) fail(static_cast<Errc>(st_code - 1), "apply_map(" + st.map + ") restatement");
  auto put_blob = [&](const char* name, const void* src, std::size_t nbytes) {
    const auto* b = static_cast<const std::uint8_t*>(src);
    s.values[name] = Blob(b, b + nbytes);
  };
  put_blob("data", buf3[0].data(), cl.n * 12);
  if (present[1]) put_blob("normal", buf3[1].data(), cl.n_normal * 12);
  if (present[2]) put_blob("color", buf3[2].data(), cl.n_color * 12);
  if (cl.intensity) put_blob("intensity", bi.data(), cl.n_intensity * 4);
  for (std::size_t e = 0; e < extra.size(); ++e)
    put_blob(extra[e].c_str(), eb[e].data(), cl.n_extra[e] * cl.extra_elem[e]);
  if (want_counts) put_blob("count", counts.data(), cl.n_counts * 4);
  return s;
}

}  // namespace

extern "C" {

// prefix_json: [{"map":..., "params":{...}, "op_id":k}, ...] applied in the
// SourceFn; graph_json holds the reference-op suffix (map nodes) to run in
// the Pipeline.  source_workers = threads for the SourceFn.
int ref_bench_composed(const char* primary, const char* graph_json, const char* prefix_json,
                       std::uint32_t repeats, const std::uint64_t* ids, std::size_t n_ids,
                       double* cost_time_s, std::uint64_t* items, std::uint64_t* batches,
                       double* avg_cpu_percent) {
  return guarded([&] {
    auto rd = std::make_shared<DatasetReader>(primary);
    auto idx = std::make_shared<IndexTable>(
        select_entries(build_index({rd->header()}), ids, n_ids));
    const json gj = json::parse(graph_json);
    PipelineGraph g = PipelineGraph::from_json(gj);
    const std::uint64_t base = gj.value("base_seed", std::uint64_t{0});
    auto steps = std::make_shared<std::vector<Step>>();
    for (const auto& o : json::parse(prefix_json))
      steps->push_back({o.at("map").get<std::string>(), o.value("params", json::object()),
                        o.at("op_id").get<std::uint64_t>()});
    SourceFn src = [rd, idx, steps, base](std::uint64_t epoch, std::uint64_t i) {
      Sample s = rd->read_sample(idx->sample_meta_list[i]);
      for (const auto& st : *steps) {
        const std::uint64_t seed = mix_seed(base, epoch, i, st.op_id);
        if (is_ref_op(st))
          s = apply_map(map_kind_from_name(st.map), st.params, std::move(s), seed);
        else
          s = orc_apply(st, std::move(s), seed);
      }
      return s;
    };
    BenchReport rep = run_benchmark(g, src, idx->size(), repeats, 50);
    *cost_time_s = rep.cost_time_s;
    *items = rep.items;
    *batches = rep.batches;
    *avg_cpu_percent = rep.avg_cpu_percent;
  });
}

}  // extern "C"

extern "C" {

// simulate_data_parallel (distributed.cpp:88-164) over the dataset's samples
// in index order; final parameters of device 0 into params (in/out).
int ref_simulate_dp(const char* primary, std::uint32_t num_devices, std::uint64_t epochs,
                    std::uint32_t per_device_batch, double* params, std::size_t dim, double lr,
                    double* max_divergence) {
  return guarded([&] {
    DatasetReader rd(primary);
    IndexTable idx = build_index({rd.header()});
    std::vector<Sample> ds;
    for (std::size_t i = 0; i < idx.size(); ++i) ds.push_back(rd.read_sample(idx.sample_meta_list[i]));
    ToyModel m;
    m.params.assign(params, params + dim);
    m.learning_rate = lr;
    SimOptions o;
    o.num_devices = num_devices;
    o.num_epochs = epochs;
    o.per_device_batch = per_device_batch;
    const SimReport r = simulate_data_parallel(ds, m, o);
    for (std::size_t j = 0; j < dim; ++j) params[j] = r.device_params[0][j];
    *max_divergence = r.max_param_divergence;
  });
}

}  // extern "C"
