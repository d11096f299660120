// gpu_pipeline.hpp — the binding a pcpipe maintainer adds to the reference
// (proj/core/include/pcpipe/gpu_pipeline.hpp; link -lpcpipe_b200).
//
// GpuPipeline is a drop-in for Pipeline over a dataset_source
// (pipeline.hpp:157-182, pcpipe_main.cpp:49-53): same graph JSON, same
// (epoch, index) seeding, same batch order, same failure contract
// (PcError(kWorkerPanic, "op <id>: ...")), batches as reference Batch objects
// in host memory.  Decode + map operators + batch assembly run on the B200
// (include/pcpipe_b200.h).  Compiled against the reference headers by
// oracle/Makefile (target `integration`) and exercised by
// integration/check_gpu_pipeline.cpp.
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "pcpipe/errors.hpp"
#include "pcpipe/pipeline.hpp"
#include "pcpipe_b200.h"

namespace pcpipe {

class GpuPipeline {
 public:
  // shard: optional entry list (e.g. one GPU's shard_index / slice shard);
  // its positions are the seed indices, like Pipeline(graph, src,
  // shard.size()) in stream_dataset (streaming.cpp:357).
  GpuPipeline(const std::string& primary, const PipelineGraph& g,
              const std::vector<std::uint64_t>* shard = nullptr, int device = 0,
              std::uint64_t epochs = 1, const std::string& extra_options = "") {
    const std::string gj = g.to_json().dump();
    // host_batches: fields arrive in pinned host memory, like the reference's Batch
    std::string opts = "{\"epochs\":" + std::to_string(epochs) + ",\"host_batches\":true";
    if (!extra_options.empty()) opts += "," + extra_options;
    opts += "}";
    check(pcp_pipeline_open(primary.c_str(), gj.c_str(), shard ? shard->data() : nullptr,
                            shard ? shard->size() : 0, device, opts.c_str(), &p_));
  }
  GpuPipeline(const GpuPipeline&) = delete;
  GpuPipeline& operator=(const GpuPipeline&) = delete;
  ~GpuPipeline() { pcp_pipeline_close(p_); }

  // Pipeline::next_batch: nullopt at the end; failures throw
  // PcError(kWorkerPanic, "op <id>: ...").
  std::optional<Batch> next_batch() {
    pcp_batch b;
    int eos = 0;
    check(pcp_pipeline_next_batch(p_, &b, &eos));
    if (eos) return std::nullopt;
    Batch out;
    out.epoch = b.epoch;
    out.batch_index = b.batch_index;
    out.samples.resize(b.n_samples);
    for (std::uint32_t f = 0; f < b.n_fields; ++f) {  // already in host memory
      const pcp_field& fd = b.fields[f];
      for (std::uint32_t s = 0; s < b.n_samples; ++s) {
        const std::uint8_t* p = fd.h_ptr + fd.h_offsets[s];
        const std::size_t n = fd.h_offsets[s + 1] - fd.h_offsets[s];
        out.samples[s].values[fd.name] = to_value(fd.kind, p, n);
      }
    }
    return out;
  }

  // Pipeline::update_op_config analogue for the device knobs.
  void update_config(const std::string& json) { check(pcp_pipeline_update_config(p_, json.c_str())); }
  std::string metrics_json() const { return pcp_pipeline_metrics(p_); }

 private:
  // FieldKind (format.hpp:25) -> Value (format.hpp:52-54)
  static Value to_value(std::int32_t kind, const std::uint8_t* p, std::size_t n) {
    auto vec = [&](auto tag) {
      using T = decltype(tag);
      std::vector<T> v(n / sizeof(T));
      if (n) std::memcpy(v.data(), p, v.size() * sizeof(T));
      return Value(std::move(v));
    };
    switch (kind) {
      case 0: return Value(Blob(p, p + n));
      case 1: return vec(std::int32_t{});
      case 2: return vec(std::int64_t{});
      case 3: return vec(float{});
      case 4: return vec(double{});
      default: return Value(std::string(reinterpret_cast<const char*>(p), n));
    }
  }
  // pcp_last_error() reads like PcError::what() ("<Errc name>: <message>");
  // rebuild the PcError from the message part.
  static void check(int st) {
    if (!st) return;
    std::string msg = pcp_last_error();
    const std::string pre = std::string(pcp_errc_name(st)) + ": ";
    if (msg.rfind(pre, 0) == 0) msg = msg.substr(pre.size());
    fail(static_cast<Errc>(st - 1), msg);
  }
  pcp_pipeline* p_ = nullptr;
};

}  // namespace pcpipe
