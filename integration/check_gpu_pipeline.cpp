// check_gpu_pipeline.cpp — the reference's pipeline order/determinism cases
// (proj/tests/test_pipeline.cpp:227-317) re-run through GpuPipeline
// (integration/gpu_pipeline.hpp) and compared with the reference Pipeline
// over dataset_source on the same .pcrecord files.  Built by oracle/Makefile
// (target `integration`, against the reference headers and the compiled
// reference sources); run by tests/test_gpu_integration.py on a B200.
// Prints [PASS]/[FAIL] per case (acceptance.cpp style); exit code = failures.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "gpu_pipeline.hpp"
#include "pcpipe/format.hpp"
#include "pcpipe/metadata.hpp"
#include "pcpipe/pipeline.hpp"

using namespace pcpipe;
namespace fs = std::filesystem;

namespace {

int failures = 0;
void report(const char* name, bool ok, const std::string& why = "") {
  std::printf("[%s] %s%s%s\n", ok ? "PASS" : "FAIL", name, ok ? "" : ": ", why.c_str());
  if (!ok) ++failures;
}

Blob coord_blob(std::size_t n, std::uint64_t seed) {  // test_util.hpp:50-58
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> u(-1.0f, 1.0f);
  std::vector<float> v(3 * n);
  for (auto& x : v) x = u(rng);
  Blob b(v.size() * 4);
  std::memcpy(b.data(), v.data(), b.size());
  return b;
}

// tagged samples (test_pipeline.cpp:26-32) written as a dataset
std::string tagged_dataset(const fs::path& dir, std::size_t n, std::uint32_t group, bool empty_at = false,
                           std::size_t bad = 0) {
  Schema schema;
  schema.fields = {{"id", FieldType{FieldKind::kInt64, {}}}, {"data", FieldType{FieldKind::kBytes, {}}}};
  std::vector<Sample> v;
  for (std::size_t i = 0; i < n; ++i) {
    Sample s;
    s.values["id"] = std::vector<std::int64_t>{static_cast<std::int64_t>(i)};
    s.values["data"] = (empty_at && i == bad) ? Blob{} : coord_blob(8 + i % 5, 131 + i);
    v.push_back(std::move(s));
  }
  fs::create_directories(dir);
  WriteOptions o;
  o.slice_count = 2;
  o.group_size = group;
  o.stem = "ds";
  write_dataset(v, schema, o, dir);
  return (dir / "ds.pcrecord").string();
}

OpNode node(std::uint32_t id, OpNode::Kind kind, std::uint32_t workers = 1) {
  OpNode n;
  n.id = id;
  n.kind = kind;
  n.num_workers = workers;
  return n;
}
OpNode map_node(std::uint32_t id, MapKind kind, std::uint32_t workers = 1) {
  OpNode n = node(id, OpNode::Kind::kMap, workers);
  n.transforms = {{kind, json::object()}};
  n.seed_op_ids = {id};
  return n;
}
PipelineGraph simple_graph(std::uint32_t batch, std::vector<OpNode> maps = {}, std::uint64_t seed = 42) {
  PipelineGraph g;
  g.nodes.push_back(node(0, OpNode::Kind::kSource));
  for (auto& m : maps) g.nodes.push_back(std::move(m));
  OpNode b = node(90, OpNode::Kind::kBatch);
  b.batch_size = batch;
  g.nodes.push_back(b);
  g.nodes.push_back(node(91, OpNode::Kind::kSink));
  g.base_seed = seed;
  return g;
}

std::vector<Batch> run_ref(const std::string& primary, const PipelineGraph& g, std::uint64_t epochs = 1) {
  auto rd = std::make_shared<DatasetReader>(primary);
  auto idx = std::make_shared<IndexTable>(build_index({rd->header()}));
  PipelineOptions opts;
  opts.epochs = epochs;
  Pipeline p(g, [rd, idx](std::uint64_t, std::uint64_t i) { return rd->read_sample(idx->sample_meta_list[i]); },
             idx->size(), opts);
  p.start();
  std::vector<Batch> out;
  while (auto b = p.next_batch()) out.push_back(std::move(*b));
  p.stop();
  return out;
}

std::vector<Batch> run_gpu(const std::string& primary, const PipelineGraph& g, std::uint64_t epochs = 1,
                           const std::string& extra = "") {
  GpuPipeline p(primary, g, nullptr, 0, epochs, extra);
  std::vector<Batch> out;
  while (auto b = p.next_batch()) out.push_back(std::move(*b));
  return out;
}

std::vector<std::int64_t> ids_of(const std::vector<Batch>& bs) {
  std::vector<std::int64_t> v;
  for (const auto& b : bs)
    for (const auto& s : b.samples) v.push_back(std::get<std::vector<std::int64_t>>(s.values.at("id"))[0]);
  return v;
}

template <typename Fn>
void run_case(const char* name, Fn&& fn) {
  try {
    fn();
  } catch (const std::exception& e) {
    report(name, false, std::string("exception: ") + e.what());
  }
}

}  // namespace

int main(int argc, char** argv) {
  const fs::path tmp = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path() / "pcp_gpu_binding";
  fs::remove_all(tmp);
  const std::string ds10 = tagged_dataset(tmp / "d10", 10, 3);
  const std::string ds50 = tagged_dataset(tmp / "d50", 50, 4);

  run_case("batches come out in dataset order", [&] {
    auto b = run_gpu(ds10, simple_graph(4));
    report("batches come out in dataset order",
           b.size() == 2 && b[0].batch_index == 0 && b[1].batch_index == 1 &&
               ids_of(b) == std::vector<std::int64_t>{0, 1, 2, 3, 4, 5, 6, 7} && b == run_ref(ds10, simple_graph(4)));
  });
  run_case("remainder batch kept when requested", [&] {
    auto g = simple_graph(4);
    g.drop_remainder = false;
    auto b = run_gpu(ds10, g);
    report("remainder batch kept when requested",
           b.size() == 3 && b[2].samples.size() == 2 && ids_of(b).size() == 10 && b == run_ref(ds10, g));
  });
  run_case("worker counts never change batch contents", [&] {
    auto mk = [](std::uint32_t w) {
      return simple_graph(5, {map_node(1, MapKind::kTranslate, w), map_node(2, MapKind::kRandomScale, w),
                              map_node(3, MapKind::kFlipYz, w)});
    };
    const auto base = run_ref(ds50, mk(1));
    bool ok = run_gpu(ds50, mk(1)) == base;
    for (std::uint32_t w : {2u, 4u, 8u}) ok = ok && run_gpu(ds50, mk(w)) == base;
    report("worker counts never change batch contents", ok);
  });
  run_case("wave sizes and slots never change batch contents", [&] {
    auto g = simple_graph(5, {map_node(1, MapKind::kNormalize), map_node(2, MapKind::kRandomScale)});
    const auto base = run_ref(ds50, g);
    bool ok = true;
    for (const char* o : {"\"wave_batches\":1,\"slots\":2", "\"wave_batches\":3,\"slots\":5",
                          "\"resident\":false", "\"stream\":true,\"wave_batches\":2"})
      ok = ok && run_gpu(ds50, g, 1, o) == base;
    report("wave sizes and slots never change batch contents", ok);
  });
  run_case("fused and unfused pipelines produce identical batches", [&] {
    auto g = simple_graph(4, {map_node(1, MapKind::kTranslate, 2), map_node(2, MapKind::kRandomScale, 3)});
    const auto plain = run_gpu(ds50, g);
    report("fused and unfused pipelines produce identical batches",
           plain == run_gpu(ds50, fuse_maps(g)) && plain == run_ref(ds50, g));
  });
  run_case("two runs with the same seed are bit-identical", [&] {
    auto g = simple_graph(4, {map_node(1, MapKind::kRotate, 4)});
    report("two runs with the same seed are bit-identical", run_gpu(ds50, g) == run_gpu(ds50, g));
  });
  run_case("multiple epochs emit every epoch in order", [&] {
    auto b = run_gpu(ds10, simple_graph(5), 3);
    bool ok = b.size() == 6;
    for (std::size_t i = 0; ok && i < b.size(); ++i) ok = b[i].epoch == i / 2 && b[i].batch_index == i % 2;
    const auto one = run_gpu(ds10, simple_graph(5));
    ok = ok && std::vector<Batch>(b.begin(), b.begin() + 2) == one && b == run_ref(ds10, simple_graph(5), 3);
    report("multiple epochs emit every epoch in order", ok);
  });
  run_case("worker failure surfaces as WorkerPanic naming the op", [&] {
    const std::string bad = tagged_dataset(tmp / "bad", 12, 4, true, 6);
    auto g = simple_graph(4, {map_node(7, MapKind::kNormalize)});
    std::string ref_msg, gpu_msg;
    Errc ref_code = Errc::kIoFailure, gpu_code = Errc::kIoFailure;
    std::size_t ref_n = 0, gpu_n = 0;
    try {
      auto rd = std::make_shared<DatasetReader>(bad);
      auto idx = std::make_shared<IndexTable>(build_index({rd->header()}));
      Pipeline p(g, [rd, idx](std::uint64_t, std::uint64_t i) { return rd->read_sample(idx->sample_meta_list[i]); },
                 idx->size());
      p.start();
      while (p.next_batch()) ++ref_n;
    } catch (const PcError& e) {
      ref_code = e.code();
      ref_msg = e.what();
    }
    try {
      GpuPipeline p(bad, g);
      while (p.next_batch()) ++gpu_n;
    } catch (const PcError& e) {
      gpu_code = e.code();
      gpu_msg = e.what();
    }
    report("worker failure surfaces as WorkerPanic naming the op",
           ref_code == Errc::kWorkerPanic && gpu_code == Errc::kWorkerPanic && gpu_n == 1 &&
               gpu_msg == ref_msg,
           "ref: " + ref_msg + " | gpu: " + gpu_msg + " after " + std::to_string(gpu_n) + " batches");
  });
  run_case("metrics reflect emitted batches", [&] {
    GpuPipeline p(ds50, simple_graph(4, {map_node(1, MapKind::kNormalize, 2)}));
    std::size_t n = 0;
    while (p.next_batch()) ++n;
    const json m = json::parse(p.metrics_json());
    report("metrics reflect emitted batches",
           m.at("batches_emitted").get<std::size_t>() == n && m.at("items_emitted").get<std::size_t>() == 4 * n &&
               m.at("ops").size() == 3);
  });
  fs::remove_all(tmp);
  std::printf("%d failure(s)\n", failures);
  return failures;
}
