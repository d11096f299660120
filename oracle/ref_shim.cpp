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
#include <vector>

#include "pcpipe/bench.hpp"
#include "pcpipe/distributed.hpp"
#include "pcpipe/errors.hpp"
#include "pcpipe/format.hpp"
#include "pcpipe/lz4_block.hpp"
#include "pcpipe/metadata.hpp"
#include "pcpipe/pipeline.hpp"
#include "pcpipe/transforms.hpp"

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
