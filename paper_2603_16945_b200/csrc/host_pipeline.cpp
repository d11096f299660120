// host_pipeline.cpp — the B200 replacement for the reference Pipeline on the
// PcRecord → batch path, and the extern "C" boundary (include/pcpipe_b200.h).
//
// Reference behaviour kept (proj/core/src/pipeline.cpp):
//   * graph JSON + validation (PipelineGraph::from_json / validate, :40-146),
//     fused map nodes expanded with their original op ids for seeding;
//   * Item (epoch, index = position within the epoch) drives mix_seed
//     (:442-462,474-476); output order = walk order; batch_index resets per
//     epoch; drop_remainder (:567-613);
//   * failures surface from next_batch as WorkerPanic "op <id>: ..." (:677-689).
// Replaced: the thread/Connector/BoundedQueue machinery.  Work is cut into
// waves of whole batches; each wave is one set of kernel launches on one
// CUDA stream (copy → CRC → page decode → record parse → per-sample
// interpreter), and the next wave is launched before the current one is
// served, so host staging, H2D copies and compute overlap.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pcpipe_b200.h"
#include "host_format.h"
#include "json.hpp"
#include "kernels.h"
#include "voxel_wave.h"

namespace pcp {

using json = nlohmann::ordered_json;
namespace fs = std::filesystem;

namespace {

thread_local std::string g_err;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kIoFailure, std::string("CUDA ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return kOk;
  } catch (const Fail& f) {
    g_err = std::string(errc_name(f.code)) + ": " + f.what();
    return f.code;
  } catch (const std::exception& e) {
    g_err = std::string("WorkerPanic: ") + e.what();
    return kWorkerPanic;
  }
}

int require_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    fail(kIoFailure, "no CUDA device: the B200 path has no CPU fallback");
  if (device < 0 || device >= n) fail(kOutOfBounds, "device index out of range");
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, device));
  if (p.major != 10) fail(kIoFailure, "device is not sm_100 (B200); this build targets sm_100a only");
  CK(cudaSetDevice(device));
  return p.multiProcessorCount;
}

// ---------------------------------------------------------------- device memory
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t want) {
    if (want <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    want = std::max<size_t>(want, 256);
    CK(cudaMalloc(&p, want));
    n = want;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct HostBuf {  // pinned
  void* p = nullptr;
  size_t n = 0;
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t want) {
    if (want <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    want = std::max<size_t>(want, 256);
    CK(cudaMallocHost(&p, want));
    n = want;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// Process-wide pool of pinned host blocks (power-of-two sizes): a pipeline
// reopened on the same process (e.g. a new epoch range) reuses the blocks
// instead of paying cudaMallocHost again.
struct PinnedPool {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;
  static PinnedPool& get() {
    static PinnedPool* p = new PinnedPool;  // never destroyed: blocks outlive atexit order
    return *p;
  }
  void* take(size_t want, size_t* got) {
    size_t cls = 4096;
    while (cls < want) cls <<= 1;
    {
      std::lock_guard<std::mutex> l(mu);
      auto it = free_blocks.lower_bound(cls);
      if (it != free_blocks.end() && it->first <= 2 * cls) {
        void* q = it->second;
        *got = it->first;
        free_blocks.erase(it);
        return q;
      }
    }
    void* q = nullptr;
    CK(cudaMallocHost(&q, cls));
    *got = cls;
    return q;
  }
  void give(void* q, size_t n) {
    std::lock_guard<std::mutex> l(mu);
    free_blocks.emplace(n, q);
  }
};

struct PooledHostBuf {
  void* p = nullptr;
  size_t n = 0;
  ~PooledHostBuf() {
    if (p) PinnedPool::get().give(p, n);
  }
  void ensure(size_t want) {
    if (want <= n) return;
    if (p) PinnedPool::get().give(p, n);
    p = PinnedPool::get().take(want, &n);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

inline uint64_t align16(uint64_t v) { return (v + 15) & ~uint64_t(15); }
inline uint64_t align4(uint64_t v) { return (v + 3) & ~uint64_t(3); }

// ---------------------------------------------------------------- graph
struct MapStep {
  int32_t kind;
  uint32_t node_id;     // the (possibly fused) map node, for error messages
  uint32_t seed_op_id;  // original op id (fuse_maps, pipeline.cpp:148-168)
  json params;
};

struct Graph {
  uint64_t base_seed = 0;
  bool drop_remainder = true;
  uint32_t source_id = 0, batch_id = 0;
  uint32_t batch_size = 1;
  std::vector<MapStep> maps;
};

int32_t map_kind_from_name(const std::string& n) {  // transforms.cpp:54-66 + App. C
  static const std::map<std::string, int32_t> m = {
      {"normalize", kNormalize}, {"translate", kTranslate}, {"jitter", kJitter},
      {"rotate", kRotate}, {"random_scale", kRandomScale}, {"flip_yz", kFlipYz},
      {"color_augment", kColorAugment}, {"random_crop", kRandomCrop},
      {"downsample", kDownsample}, {"fps", kFps}, {"voxel", kVoxel},
      {"grid_subsample", kVoxel}, {"range_crop", kRangeCrop}};
  auto it = m.find(n);
  if (it == m.end()) fail(kUnknownOp, "unknown map '" + n + "'");
  return it->second;
}

Graph parse_graph(const std::string& text) {
  json j = json::parse(text, nullptr, false);
  if (j.is_discarded()) fail(kUnknownOp, "graph is not valid JSON");
  Graph g;
  struct Node {
    uint32_t id;
    std::string kind;
    uint32_t workers, queue, batch;
    std::vector<MapStep> steps;
  };
  std::vector<Node> nodes;
  try {
    g.base_seed = j.value("base_seed", uint64_t{0});
    g.drop_remainder = j.value("drop_remainder", true);
    for (const auto& o : j.at("ops")) {
      Node n;
      n.id = o.at("id").get<uint32_t>();
      n.kind = o.at("kind").get<std::string>();
      if (n.kind != "source" && n.kind != "map" && n.kind != "batch" && n.kind != "sink")
        fail(kUnknownOp, "op kind '" + n.kind + "'");
      n.workers = o.value("num_workers", 1u);
      n.queue = o.value("queue_capacity", 8u);
      n.batch = o.value("batch_size", 1u);
      if (n.kind == "map") {
        if (o.contains("fused")) {
          for (const auto& f : o["fused"]) {
            n.steps.push_back({map_kind_from_name(f.at("map").get<std::string>()), n.id,
                               f.at("op_id").get<uint32_t>(), f.value("params", json::object())});
            if (f.at("map").get<std::string>() == "grid_subsample" &&
                n.steps.back().params.is_object() && !n.steps.back().params.contains("counts"))
              n.steps.back().params["counts"] = false;
          }
        } else {
          n.steps.push_back({map_kind_from_name(o.at("map").get<std::string>()), n.id, n.id,
                             o.value("params", json::object())});
          if (o.at("map").get<std::string>() == "grid_subsample" && n.steps.back().params.is_object() &&
              !n.steps.back().params.contains("counts"))
            n.steps.back().params["counts"] = false;
        }
      }
      nodes.push_back(std::move(n));
    }
  } catch (const json::exception& e) {
    fail(kUnknownOp, std::string("malformed graph: ") + e.what());
  }
  // PipelineGraph::validate (:40-80)
  if (nodes.size() < 3) fail(kUnknownOp, "graph needs source, batch, sink");
  if (nodes.front().kind != "source") fail(kUnknownOp, "first node must be a source");
  if (nodes.back().kind != "sink") fail(kUnknownOp, "last node must be a sink");
  bool batch_seen = false;
  for (size_t i = 0; i < nodes.size(); ++i) {
    const auto& n = nodes[i];
    for (size_t k = 0; k < i; ++k)
      if (nodes[k].id == n.id) fail(kUnknownOp, "duplicate op id");
    if (n.workers < 1 || n.queue < 1) fail(kOutOfBounds, "workers and queue capacity must be >= 1");
    if (n.kind == "source" && i != 0) fail(kUnknownOp, "source must come first");
    if (n.kind == "map") {
      if (batch_seen) fail(kUnknownOp, "map after batch");
      if (n.steps.empty()) fail(kUnknownOp, "map without transform");
      for (const auto& s : n.steps) g.maps.push_back(s);
    }
    if (n.kind == "batch") {
      if (batch_seen) fail(kUnknownOp, "more than one batch node");
      if (n.batch < 1) fail(kOutOfBounds, "batch_size must be >= 1");
      batch_seen = true;
      g.batch_size = n.batch;
      g.batch_id = n.id;
    }
    if (n.kind == "sink" && i + 1 != nodes.size()) fail(kUnknownOp, "sink must come last");
  }
  if (!batch_seen) fail(kUnknownOp, "graph needs a batch node");
  g.source_id = nodes.front().id;
  if (g.maps.size() > (size_t)kMaxOps) fail(kOutOfBounds, "too many map transforms for one stage");
  return g;
}

// Map params JSON → OpDesc (transforms.cpp:103-113,171-172,273 + App. C).
// busy_us / sleep_us are CPU cost-injection knobs of the reference
// (transforms.cpp:103-113); they have no meaning on the device and are ignored.
template <typename IndexOf>
void parse_op_params(OpDesc& op, const json& p, IndexOf bytes_index_of) {
  if (!p.is_object() && !p.is_null()) fail(kUnknownOp, "map params must be an object");
  try {
    if (p.is_object()) {
      if (p.contains("theta")) {
        op.has_theta = 1;
        op.theta = p["theta"].get<float>();
      }
      if (p.contains("num_points")) op.num_points = p["num_points"].get<int64_t>();
      if (p.contains("gather")) {
        for (const auto& nm : p["gather"]) {
          const int bi = bytes_index_of(nm.get<std::string>());
          if (bi < 0) fail(kMissingField, "gather field '" + nm.get<std::string>() + "' is not a bytes field");
          op.gather_mask |= 1u << bi;
        }
      }
      if (p.contains("voxel_size")) op.voxel = p["voxel_size"].get<float>();
      if (p.contains("origin")) {
        op.has_origin = 1;
        for (int i = 0; i < 3; ++i) op.origin[i] = p["origin"][i].get<float>();
      }
      op.counts = p.value("counts", op.kind == kVoxel ? 1 : 0);
      if (p.contains("lo"))
        for (int i = 0; i < 3; ++i) op.lo[i] = p["lo"][i].get<float>();
      if (p.contains("hi"))
        for (int i = 0; i < 3; ++i) op.hi[i] = p["hi"][i].get<float>();
    }
  } catch (const json::exception& e) {
    fail(kOutOfBounds, std::string("bad map params: ") + e.what());
  }
  if ((op.kind == kDownsample || op.kind == kFps) && op.num_points <= 0)
    fail(kOutOfBounds, "num_points must be positive");
  if (op.kind == kVoxel && !(op.voxel > 0.0f)) fail(kOutOfBounds, "voxel_size must be positive");
}

// Per-CTA buffer plan of k_cloud / k_apply_set (buffer ids in WaveArgs):
// sizes follow what the op chain can need; shared memory is filled greedily
// in priority order (coordinates first), everything else goes to the per-CTA
// global slab (a.gscratch_per_cta).  Returns the shared bytes used.
// Cluster FPS plan: a static bound on the points any FPS op
// sees — the cloud capacity, or T after a downsample / M after an FPS (both
// leave exactly that many points; crops and voxel never grow a cloud).  A
// bound above one CTA's register capacity (kFpsRegPts x threads) splits the
// cloud over a thread-block cluster of up to 8 CTAs; beyond that the
// global-memory FPS path runs in one CTA.
void plan_fps_cluster(WaveArgs& a, uint32_t threads) {
  uint64_t bound = a.cap_points, need = 0;
  for (int k = 0; k < a.n_ops; ++k) {
    const OpDesc& op = a.ops[k];
    if (op.kind == kFps) {
      need = std::max(need, bound);
      bound = (uint64_t)std::max<int64_t>(op.num_points, 0);
    } else if (op.kind == kDownsample) {
      bound = (uint64_t)std::max<int64_t>(op.num_points, 0);
    }
  }
  const uint64_t per_cta = (uint64_t)kFpsRegPts * threads;
  a.fps_cluster = 1;
  a.fps_slice_pts = 0;
  if (need > per_cta) {
    const uint64_t C = (need + per_cta - 1) / per_cta;
    if (C <= 8) {
      a.fps_cluster = (uint32_t)C;
      a.fps_slice_pts = (uint32_t)((need + C - 1) / C);
    }
  }
}

size_t plan_buffers(WaveArgs& a, bool want_staging, size_t smem_budget) {
  uint64_t T = 0, M = 0;
  bool ds = false, fps = false, crop = false, vox = false;
  for (int k = 0; k < a.n_ops; ++k) {
    const OpDesc& op = a.ops[k];
    if (op.kind == kDownsample) ds = true, T = std::max<uint64_t>(T, (uint64_t)op.num_points);
    if (op.kind == kFps) fps = true, M = std::max<uint64_t>(M, (uint64_t)op.num_points);
    if (op.kind == kRandomCrop || op.kind == kRangeCrop) crop = true;
    if (op.kind == kVoxel) vox = true;
  }
  const uint64_t cap = a.cap_points;
  const uint64_t big = (crop || vox) ? cap : 0;
  const uint64_t alt_pts = std::max({T, M, big});
  auto with = [](uint64_t b) { return b ? b + 16 : 0; };
  uint64_t* sz = a.buf_bytes;
  for (int b = 0; b < 26; ++b) sz[b] = 0;
  if (a.fps_cluster > 1) sz[24] = kFpsMailBytes + 12ull * a.fps_slice_pts + 16;
  if (vox) sz[25] = kSortScratchBytes;
  sz[0] = want_staging ? (uint64_t)a.max_blob + 64 : 0;
  sz[1] = 4 * std::max<uint64_t>({T, M, big, 1}) + 16;
  sz[2] = with(4 * ((ds || fps || vox) ? cap : 0));
  sz[3] = with(4 * std::max<uint64_t>(ds ? T : 0, vox ? cap : 0));
  sz[4] = with(4 * (ds ? T : 0));
  for (int f = 0; f < a.n_bytes_fields; ++f) {
    if (!((a.tracked_mask >> f) & 1u)) continue;
    sz[5 + f] = cap * a.field_cap[f] + 16;
    sz[13 + f] = with(alt_pts * a.field_cap[f]);
  }
  if (vox) {
    sz[21] = sz[22] = 8 * cap + 16;
    sz[23] = 4 * cap + 16;
  }
  std::vector<int> order;
  if (sz[24]) order.push_back(24);  // cluster-FPS slice + mailbox first (latency-critical)
  if (sz[25]) order.push_back(25);  // voxel sort scratch: smem atomics / per-warp counts
  const int rd = a.role_data;
  if (rd >= 0) order.push_back(5 + rd);
  for (int b : {1, 3, 4}) order.push_back(b);
  if (rd >= 0) order.push_back(13 + rd);
  order.push_back(2);
  for (int f = 0; f < kMaxBytesFields; ++f)
    if (f != rd) order.push_back(5 + f);
  for (int f = 0; f < kMaxBytesFields; ++f)
    if (f != rd) order.push_back(13 + f);
  for (int b : {21, 22, 23, 0}) order.push_back(b);
  auto rnd = [](uint64_t v) { return (v + 127) & ~uint64_t(127); };
  size_t used = 0;
  uint64_t gbytes = 0;
  a.buf_smem_mask = 0;
  for (int b : order) {
    if (!sz[b]) continue;
    if (used + rnd(sz[b]) <= smem_budget) {
      used += rnd(sz[b]);
      a.buf_smem_mask |= 1u << b;
    } else if (b == 0) {
      sz[0] = 0;  // no staging: decode reads the blob from global memory
    } else {
      gbytes += rnd(sz[b]);
    }
  }
  a.smem_mode = a.buf_smem_mask ? 1 : 0;
  a.gscratch_per_cta = gbytes;
  return used;
}

// Per-device state for the stateless entry points (codec + operator API).
struct DeviceCtx {
  int sms = 0;
  DevBuf shift, scratch;
};
DeviceCtx& device_ctx(cudaStream_t st) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<DeviceCtx>> ctxs;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto& c = ctxs[dev];
  if (!c) {
    c = std::make_unique<DeviceCtx>();
    c->sms = require_device(dev);
    upload_x2n(st);
    std::vector<uint32_t> shift(kShiftTabWords);
    build_shift_table(shift.data());
    c->shift.ensure(shift.size() * 4);
    CK(cudaMemcpy(c->shift.p, shift.data(), shift.size() * 4, cudaMemcpyHostToDevice));
  }
  return *c;
}

// ---------------------------------------------------------------- pipeline
struct OutField {
  std::string name;
  int32_t kind;        // value kind of the batch field
  int32_t schema_idx;  // schema field, or -1 for synthesized fields
  uint64_t stride;     // slot bytes per sample
  bool varlen;         // bytes / string: per-sample lengths may differ (CSR)
};

struct Wave {
  uint64_t epoch = 0;
  uint64_t pos0 = 0, n = 0;  // positions [pos0, pos0+n) of the epoch
  uint64_t first_batch = 0;  // batch index of the wave's first batch
  uint32_t n_batches = 0;
  bool launched = false;
  cudaStream_t stream = nullptr;  // one stream per slot: consecutive waves overlap
  cudaEvent_t done = nullptr, k0 = nullptr, k1 = nullptr, d0 = nullptr, d1 = nullptr;
  cudaEvent_t c0 = nullptr, c1 = nullptr, s0 = nullptr, s1 = nullptr;  // CRC windows, wave CSR
  uint64_t crc_alg_bytes = 0;     // payload bytes k_crc_windows reads
  uint64_t vx_alg_bytes = 0;      // decoded tracked-field bytes the vx stage reads
  cudaEvent_t h0 = nullptr, h1 = nullptr;  // staging copies (timeline diagnostics)
  cudaEvent_t served = nullptr;  // serve stream passed this wave's last batch (user copies enqueued)
  uint64_t decode_alg_bytes = 0;  // payload + raw bytes of the pages k_page_decode handles
  DevBuf gscratch;                // k_cloud global slab (smem_mode 0), per slot
  // device
  DevBuf bytes_stage, raw, tables, outs, compact, lz4_scratch, lz4_timing;
  DevBuf handoff;  // chain split: the clouds between launches (decoded clouds A for the vx stage)
  DevBuf handoff_b;  // vx stage output (voxelized clouds B)
  DevBuf vx_cl, vx_tiles, vx_cnt, vx_w0, vx_w1;  // vx stage scratch
  DevBuf vx_bt, vx_bcnt, vx_boff, vx_items, vx_T;  // vx bucket mode
  DevBuf pj_ptr, pj_changed, pj_flags;  // LZ4 phase 4 by pointer jumping: source per raw byte, round / block flags
  cudaEvent_t v0 = nullptr, v1 = nullptr;        // vx stage
  DevBuf mt_pre;   // pre-seeded MT19937-64 states [n][n_rng][312] (k_seed_states)
  uint32_t n_todo = 0;
  HostBuf h_tables, h_res;
  HostBuf h_stage;  // option "stream": the wave's page runs read from the slice files
  std::vector<uint64_t> out_base;  // per output field: offset in outs (and in compact)
  // results (pinned, filled by D2H)
  int32_t* h_status = nullptr;
  int32_t* h_op = nullptr;
  int32_t* h_where = nullptr;
  uint64_t* h_len = nullptr;
  uint64_t* h_woff = nullptr;   // [n_var][n+1] sample byte offsets of varlen fields (k_wave_offsets)
  uint32_t* h_dense = nullptr;  // [n_out] every sample fills its slot
  uint64_t staged = 0;          // host_batches: samples [0, staged) are in h_out
  uint64_t in_payload_bytes = 0, in_points = 0;
  std::vector<std::vector<uint64_t>> offsets;  // per field, for the served batch
  // host_batches: the whole wave's batch fields in pinned host memory
  PooledHostBuf h_out;
  std::vector<uint64_t> h_base;                 // per field: offset in h_out
  cudaEvent_t host_ready = nullptr;
};

}  // namespace

struct Pipeline {
  int device = 0, sms = 0;
  Graph g;
  Header h;
  std::string dir;
  std::vector<Entry> index, walk;
  bool resident = true;
  uint32_t wave_batches = 0;
  bool host_batches = false;  // deliver batches in pinned host memory (one D2H per field per wave)
  uint32_t n_slots = 4;  // wave slots (streams): n_slots - 1 waves in flight while one is served
  bool slots_set = false;
  uint64_t epochs = 1;
  bool force_serial_fy = false;
  bool lz4_timing = std::getenv("PCP_LZ4_TIMING") != nullptr;
  bool op_timing = std::getenv("PCP_OP_TIMING") != nullptr;  // per-op SM cycles (diagnostics)
  bool no_fused_crc = std::getenv("PCP_NO_FUSED_CRC") != nullptr;  // experiment switch
  bool no_preseed = std::getenv("PCP_NO_PRESEED") != nullptr;  // experiment switch: seed MT in k_cloud
  DevBuf d_op_cycles;
  std::vector<double> lz4_phase_cycles = std::vector<double>(4, 0.0);
  cudaStream_t stream = nullptr;        // wave compute (copies + kernels)
  cudaStream_t serve_stream = nullptr;  // batch views: compaction, user D2H
  // byte store: all slice data areas, 16-B aligned, 64 B slack each side
  std::vector<uint64_t> slice_base;  // ~0: slice not loaded (outside the walk)
  std::vector<uint64_t> slice_len, slice_file_off;
  std::vector<int> slice_fd;
  uint64_t loaded_bytes = 0;  // slice bytes read into pinned memory at open
  std::thread reader;
  std::mutex rd_mu;
  std::condition_variable rd_cv;
  int64_t ready_upto = -1, launched_upto = -1;
  bool rd_stop = false, rd_failed = false;
  std::string rd_err;
  uint64_t read_bytes = 0;
  double read_wait_ms = 0;
  // option "stream": no byte store; each wave's pages are read from the slice
  // files by reader threads into the slot's pinned buffer ahead of its launch
  // (read → H2D → decode → transform → batch all overlap across waves)
  bool stream_files = false;
  uint32_t reader_threads = 8;
  uint64_t store_bytes = 0;
  DevBuf d_store;
  HostBuf h_store;
  DevBuf d_shift, d_gscratch;
  // page heads: [group] -> scalar, block
  std::vector<PageHead> scalar_head, block_head;
  bool block_tiles_payload_ok = true;
  uint64_t block_pages_lz4 = 0;
  // schema / outputs
  std::vector<int32_t> bytes_fields;  // schema index per bytes field
  std::vector<OutField> outs;
  std::vector<int32_t> var_index;  // batch field -> varlen slot (or -1)
  uint32_t n_var = 0;
  WaveArgs proto{};
  int threads = 512, grid = 0, grid_pre = 0;
  size_t smem = 0;
  // iteration
  std::vector<Wave> slots;
  std::vector<std::pair<uint64_t, uint64_t>> plan;  // (epoch, pos0) of waves
  std::vector<uint64_t> plan_n;
  size_t next_plan = 0;  // next wave to launch
  int cur = -1;          // slot being served
  uint32_t served = 0;   // batches served from cur
  bool failed = false;
  int32_t fail_code = 0;
  std::string fail_msg;
  std::string stats_json, metrics_json;
  json pending_cfg = json::object();
  bool has_pending = false;
  uint64_t reconfigs = 0, sink_polls = 0, sink_empty_polls = 0, items_emitted = 0;
  uint32_t cur_wave_batches = 0;
  std::chrono::steady_clock::time_point t_start = std::chrono::steady_clock::now();
  // stats
  uint64_t clouds = 0, points_in = 0, payload_bytes = 0, batches = 0;
  uint64_t h2d_bytes = 0, launches = 0, alg_bytes = 0;
  double kernel_ms = 0, cloud_kernel_ms = 0, decode_kernel_ms = 0, crc_kernel_ms = 0, csr_kernel_ms = 0;
  uint64_t crc_alg_bytes = 0, csr_alg_bytes = 0;
  bool serial = false;  // option "serial": one wave in flight (non-overlapped kernel timing)
  // multi-CTA voxel stage (voxel_wave.cu) for large clouds whose chain starts
  // with [range_crop,] voxel; option "vx": false keeps it in k_cloud
  bool vx_allowed = false, vx_on = false;  // default off until it beats the one-CTA path
  uint64_t vx_min_points = 32768;
  bool vx_msd = true;  // option "vx_buckets": bucket mode of the vx stage
  // LZ4 phase 4 by page-wide pointer jumping: -1 auto (unless the block
  // pages average >= 32 samples), 0 never, 1 always (option
  // "lz4_pointer_jumping", env PCP_LZ4_PJ)
  int lz4_pj = std::getenv("PCP_LZ4_PJ") ? std::atoi(std::getenv("PCP_LZ4_PJ")) : -1;
  uint64_t lz4_pj_waves = 0;  // waves whose LZ4 phase 4 ran as pointer jumping
  bool stagger_start = !(std::getenv("PCP_STAGGER") && std::atoi(std::getenv("PCP_STAGGER")) == 0);
  uint64_t waves_launched_total = 0;
  cudaEvent_t first_k1 = nullptr;  // the first wave's end-of-chain event (slot-owned)
  VxArgs vx_proto{};
  double vx_kernel_ms = 0;
  uint64_t vx_alg_bytes = 0;
  double host_launch_ms = 0, host_wait_ms = 0;  // host-side wall time (diagnostics)
  bool timeline_on = false;
  cudaEvent_t t_open = nullptr;
  std::chrono::steady_clock::time_point host_open;
  std::vector<std::vector<double>> timeline;
  uint64_t decode_alg_bytes = 0;
  uint64_t d2h_bytes = 0;  // host_batches: batch bytes copied to host
  uint32_t waves_done = 0;

  void create_slot(Wave& w) {
    CK(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
    for (size_t pi = 0; pi < plan.size() && plan[pi].first == plan[next_plan < plan.size() ? next_plan : 0].first;
         ++pi)
      if (pi >= next_plan) launch(w, pi, true);  // pre-size for the waves still to come
    if (proto.gscratch_per_cta) w.gscratch.ensure(proto.gscratch_per_cta * std::max(grid, grid_pre));
    for (cudaEvent_t* e : {&w.done, &w.k0, &w.k1, &w.d0, &w.d1, &w.h0, &w.h1, &w.c0, &w.c1, &w.s0, &w.s1, &w.v0, &w.v1})
      CK(cudaEventCreate(e));
    CK(cudaEventCreateWithFlags(&w.served, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&w.host_ready, cudaEventDisableTiming));
    CK(cudaEventRecord(w.served, serve_stream));
  }

  static void destroy_slot(Wave& w) {
    if (w.stream) cudaStreamDestroy(w.stream);
    for (cudaEvent_t e : {w.done, w.k0, w.k1, w.d0, w.d1, w.h0, w.h1, w.c0, w.c1, w.s0, w.s1, w.v0, w.v1,
                          w.served, w.host_ready})
      if (e) cudaEventDestroy(e);
    w.stream = nullptr;
  }

  ~Pipeline() {
    if (reader.joinable()) {
      {
        std::lock_guard<std::mutex> lk(rd_mu);
        rd_stop = true;
      }
      rd_cv.notify_all();
      reader.join();
    }
    for (int fd : slice_fd)
      if (fd >= 0) ::close(fd);
    for (auto& w : slots) destroy_slot(w);
    if (t_open) cudaEventDestroy(t_open);
    if (stream) cudaStreamDestroy(stream);
    if (serve_stream) cudaStreamDestroy(serve_stream);
  }

  // Caller-supplied pages (pcp_pipeline_open_source): the SourceFn analogue.
  pcp_page_source_fn src_read = nullptr;
  pcp_wave_done_fn src_done = nullptr;
  void* src_user = nullptr;
  const std::vector<uint8_t>* src_header = nullptr;

  void open(const std::string& primary, const std::string& graph_json, const uint64_t* ids,
            uint64_t n_ids, int dev, const std::string& options) {
    sms = require_device(dev);
    device = dev;
    g = parse_graph(graph_json);
    if (const char* e = std::getenv("PCP_VX")) vx_allowed = std::atoi(e) != 0;  // experiment switch
    if (!options.empty()) {
      json o = json::parse(options, nullptr, false);
      if (o.is_discarded()) fail(kOutOfBounds, "options are not valid JSON");
      epochs = o.value("epochs", uint64_t{1});
      resident = o.value("resident", true);
      wave_batches = o.value("wave_batches", 0u);
      host_batches = o.value("host_batches", false);
      if (o.contains("slots")) {
        n_slots = std::max(2u, std::min(8u, o.value("slots", n_slots)));
        slots_set = true;
      }
      force_serial_fy = o.value("force_serial_fy", false);
      serial = o.value("serial", false);
      stream_files = o.value("stream", false);
      reader_threads = std::max(1u, std::min(64u, o.value("reader_threads", reader_threads)));
      if (stream_files) resident = false;
      vx_allowed = o.value("vx", vx_allowed);
      vx_min_points = o.value("vx_min_points", vx_min_points);
      vx_msd = o.value("vx_buckets", vx_msd);
      if (o.contains("lz4_pointer_jumping")) lz4_pj = o["lz4_pointer_jumping"].get<bool>() ? 1 : 0;
    }
    if (src_header) {  // pages come from the caller: header bytes only, no files
      h = parse_header_bytes(src_header->data(), src_header->size());
      stream_files = true;
      resident = false;
    } else {
      h = read_header(primary);
      dir = fs::path(primary).parent_path().string();
    }
    index = build_index(h);
    if (ids) {
      for (uint64_t i = 0; i < n_ids; ++i) {
        if (ids[i] >= index.size()) fail(kOutOfRange, "sample id " + std::to_string(ids[i]));
        walk.push_back(index[ids[i]]);
      }
    } else {
      walk = index;
    }
    if (walk.empty()) fail(kEmptyDataset, "no samples");
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&serve_stream, cudaStreamNonBlocking));
    load_store();
    plan_schema();
    if (const char* e = std::getenv("PCP_WAVE_BATCHES")) wave_batches = (uint32_t)std::atoi(e);  // sweep switch
    plan_waves();
    if (vx_on) {  // k_cloud launches around the vx stage: one CTA per cloud of a wave at most
      uint64_t mx = 1;
      for (uint64_t n : plan_n) mx = std::max(mx, n);
      if (proto.fps_cluster <= 1) grid = (int)std::min<uint64_t>(grid, mx);
      grid_pre = (int)std::min<uint64_t>(std::max(grid_pre, 1), mx);
    }
    upload_x2n(stream);
    std::vector<uint32_t> shift(kShiftTabWords);
    build_shift_table(shift.data());
    d_shift.ensure(shift.size() * 4);
    CK(cudaMemcpyAsync(d_shift.p, shift.data(), shift.size() * 4, cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));
    if (const char* e = std::getenv("PCP_SLOTS")) {
      n_slots = std::max(2, std::min(8, std::atoi(e)));
      slots_set = true;
    }
    // default: 4 slots (3 waves in flight: the LZ4 match phase of one wave
    // overlaps the decode / k_cloud of the others); 5 when every cloud's
    // buffers sit in shared memory (C2 +2%, measured: tools/sweep_slots.sh),
    // fewer when the per-CTA global slabs of large-cloud chains would exceed
    // 100 GiB (S3DIS: 4 slots of 26 GB; 3-4 slots measured +3% over 2)
    if (!slots_set && !proto.gscratch_per_cta) n_slots = 5;
    if (!slots_set && proto.gscratch_per_cta)
      while (n_slots > 2 && (uint64_t)n_slots * proto.gscratch_per_cta * std::max(grid, grid_pre) > (100ull << 30))
        --n_slots;
    slots.reserve(8);  // reconfiguration resizes in place (Wave owns device buffers)
    // each slot is pre-sized for its largest wave as it is created; beyond two,
    // a slot is added only while the device keeps room for one more plus a
    // margin (quantized S3DIS: slabs + raw pages + LZ4 pointer arrays ~60 GB
    // per slot)
    size_t per_slot = 0;
    for (uint32_t k = 0; k < n_slots; ++k) {
      size_t f0 = 0, f1 = 0, tot = 0;
      CK(cudaMemGetInfo(&f0, &tot));
      if (k >= 2 && per_slot && f0 < per_slot + std::max<size_t>(8ull << 30, tot / 16)) break;
      slots.emplace_back();
      create_slot(slots.back());
      CK(cudaMemGetInfo(&f1, &tot));
      per_slot = std::max<size_t>(per_slot, f0 > f1 ? f0 - f1 : 0);
    }
    n_slots = (uint32_t)slots.size();
    t_start = std::chrono::steady_clock::now();
    if (stream_files && !plan.empty()) reader = std::thread([this] { reader_main(); });
    if (const char* e = std::getenv("PCP_TIMELINE")) timeline_on = std::atoi(e) != 0;
    if (timeline_on) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventCreate(&t_open));
      CK(cudaEventRecord(t_open, serve_stream));
      CK(cudaEventSynchronize(t_open));
      host_open = std::chrono::steady_clock::now();
    }
  }

  // Slice data areas → one byte store (HBM when resident, pinned host else,
  // nothing with "stream": pages are read from the slice files per wave).
  // Shard-local: only the slices the walk touches are read and placed
  // (a rank of an N-GPU run loads ~1/N of the dataset).
  void load_store() {
    const uint32_t ns = (uint32_t)h.slice_paths.size();
    slice_base.assign(ns, ~uint64_t(0));
    slice_len.assign(ns, 0);
    slice_file_off.assign(ns, 0);
    std::vector<char> need(ns, 0);
    for (const auto& e : walk) need[h.groups[e.group_index].slice] = 1;
    uint64_t at = 64;
    std::vector<uint64_t> extent(ns, 0);  // page-covered part of each slice data area
    for (const auto& gr : h.groups)
      extent[gr.slice] = std::max({extent[gr.slice], gr.scalar_off + gr.scalar_len, gr.block_off + gr.block_len});
    for (uint32_t s = 0; s < ns; ++s) {
      if (!need[s]) continue;
      if (src_read) {
        slice_len[s] = extent[s];
      } else {
        const fs::path p = fs::path(dir) / h.slice_paths[s];
        std::error_code ec;
        const uint64_t sz = fs::file_size(p, ec);
        if (ec) fail(kIoFailure, "cannot open slice " + h.slice_paths[s]);
        slice_file_off[s] = s == 0 ? h.header_bytes : 0;
        if (sz < slice_file_off[s]) fail(kCorruptHeader, "slice shorter than its header");
        slice_len[s] = sz - slice_file_off[s];
      }
      slice_base[s] = at;
      at = align16(at + slice_len[s]) + 64;
    }
    store_bytes = at;
    slice_fd.assign(ns, -1);
    for (uint32_t s = 0; s < ns && !src_read; ++s) {
      if (!need[s]) continue;
      slice_fd[s] = ::open((fs::path(dir) / h.slice_paths[s]).c_str(), O_RDONLY | O_CLOEXEC);
      if (slice_fd[s] < 0) fail(kIoFailure, "cannot open slice " + h.slice_paths[s]);
    }
    if (!stream_files) {
      h_store.ensure(store_bytes);
      std::memset(h_store.p, 0, store_bytes);  // slack bytes between slices read as zeros
      for (uint32_t s = 0; s < ns; ++s)
        if (need[s]) read_file(s, 0, slice_len[s], h_store.as<uint8_t>() + slice_base[s]);
      loaded_bytes = 0;
      for (uint32_t s = 0; s < ns; ++s) loaded_bytes += slice_len[s];
    }
    // page heads (EncodedPage::deserialize of both pages per group)
    scalar_head.assign(h.groups.size(), PageHead{});
    block_head.assign(h.groups.size(), PageHead{});
    for (size_t gi = 0; gi < h.groups.size(); ++gi) {
      const Group& gr = h.groups[gi];
      if (!need[gr.slice]) continue;
      const uint64_t L = slice_len[gr.slice];
      auto head = [&](uint64_t off, uint64_t len) {
        const uint64_t avail = std::min(L - std::min(off, L), len);
        uint8_t buf[kPageHeaderBytes];
        const uint8_t* ph = buf;
        if (stream_files) {
          if (avail >= kPageHeaderBytes) read_file(gr.slice, off, kPageHeaderBytes, buf);
        } else {
          ph = h_store.as<uint8_t>() + slice_base[gr.slice] + off;
        }
        return parse_page_head(ph, avail);
      };
      scalar_head[gi] = head(gr.scalar_off, gr.scalar_len);
      block_head[gi] = head(gr.block_off, gr.block_len);
      if (block_head[gi].flags & kFlagOuterLz4) ++block_pages_lz4;
    }
    if (resident) {
      d_store.ensure(store_bytes);
      CK(cudaMemcpyAsync(d_store.p, h_store.p, store_bytes, cudaMemcpyHostToDevice, stream));
      CK(cudaStreamSynchronize(stream));
    }
  }

  // pread of [off, off+len) of slice s's data area (all bytes or kIoFailure).
  void read_file(uint32_t s, uint64_t off, uint64_t len, uint8_t* dst) const {
    if (src_read) {  // caller-supplied pages (may block until the slice is present)
      const int st = src_read(src_user, s, off, len, dst);
      if (st) fail(st, "page source failed for slice " + std::to_string(s));
      return;
    }
    uint64_t done = 0;
    while (done < len) {
      const ssize_t r = ::pread(slice_fd[s], dst + done, len - done, (off_t)(slice_file_off[s] + off + done));
      if (r <= 0) fail(kIoFailure, "short read of " + h.slice_paths[s]);
      done += (uint64_t)r;
    }
  }

  // Store range [lo, lo+len) → dst, from the slice files: each slice's part
  // by pread, the slack between slices as zeros.
  void read_store_range(uint64_t lo, uint64_t len, uint8_t* dst) const {
    std::memset(dst, 0, len);
    for (uint32_t s = 0; s < slice_base.size(); ++s) {
      if (slice_base[s] == ~uint64_t(0)) continue;
      const uint64_t a = std::max(lo, slice_base[s]), b = std::min(lo + len, slice_base[s] + slice_len[s]);
      if (a < b) read_file(s, a - slice_base[s], b - a, dst + (a - lo));
    }
  }

  int bytes_index_of(const std::string& name) const {
    for (size_t k = 0; k < bytes_fields.size(); ++k)
      if (h.schema[bytes_fields[k]].name == name) return (int)k;
    return -1;
  }

  void plan_schema() {
    WaveArgs& a = proto;
    std::memset(&a, 0, sizeof(a));
    a.neg_zero = -0.0f;
    if (h.schema.size() > (size_t)kMaxFields) fail(kOutOfBounds, "too many schema fields");
    a.n_fields = (int32_t)h.schema.size();
    for (size_t f = 0; f < h.schema.size(); ++f) {
      a.fields[f].kind = h.schema[f].kind;
      a.fields[f].elems = h.schema[f].elems();
      a.fields[f].bytes_index = -1;
      if (h.schema[f].kind == kBytes) {
        a.fields[f].bytes_index = (int32_t)bytes_fields.size();
        bytes_fields.push_back((int32_t)f);
      }
    }
    if (bytes_fields.size() > (size_t)kMaxBytesFields) fail(kOutOfBounds, "too many bytes fields");
    a.n_bytes_fields = (int32_t)bytes_fields.size();
    a.role_data = bytes_index_of("data");
    a.role_normal = bytes_index_of("normal");
    a.role_color = bytes_index_of("color");
    a.role_intensity = bytes_index_of("intensity");
    // ops
    a.n_ops = (int32_t)g.maps.size();
    a.base_seed = g.base_seed;
    // RNG ops get a pre-seeded MT state per sample (k_seed_states)
    a.n_rng = 0;
    for (size_t k = 0; k < g.maps.size(); ++k) {
      const int kd = g.maps[k].kind;
      const bool rng_op = kd == kTranslate || kd == kJitter || kd == kRotate || kd == kRandomScale ||
                          kd == kFlipYz || kd == kColorAugment || kd == kRandomCrop || kd == kDownsample;
      a.rng_slot[k] = rng_op && !no_preseed ? (int8_t)a.n_rng++ : (int8_t)-1;
    }
    uint32_t gather_all = 0;
    uint64_t max_target = 0;
    for (size_t k = 0; k < g.maps.size(); ++k) {
      OpDesc& op = a.ops[k];
      const MapStep& m = g.maps[k];
      op.kind = m.kind;
      op.seed_op_id = m.seed_op_id;
      parse_op_params(op, m.params, [&](const std::string& nm) { return bytes_index_of(nm); });
      gather_all |= op.gather_mask;
      max_target = std::max<uint64_t>(max_target, op.num_points > 0 ? (uint64_t)op.num_points : 0);
    }
    // tracked fields: point-cloud roles + gathered extras (only with ops)
    uint32_t tracked = 0;
    if (a.n_ops) {
      for (int r : {a.role_data, a.role_normal, a.role_color, a.role_intensity})
        if (r >= 0) tracked |= 1u << r;
      tracked |= gather_all;
    }
    a.tracked_mask = tracked;
    // capacities from the header's blob lengths
    std::vector<uint64_t> max_len(bytes_fields.size(), 0);
    uint64_t max_blob = 0, max_pts = 0;
    std::vector<uint32_t> ext_elem(bytes_fields.size(), 1);
    for (const auto& gr : h.groups)
      for (uint32_t r = 0; r < gr.sample_count; ++r) {
        const auto& L = gr.blob_lens[r];
        max_blob = std::max<uint64_t>(max_blob, gr.blob_ranges[r][1] - gr.blob_ranges[r][0]);
        const uint64_t nd = (a.role_data >= 0 && a.role_data < (int)L.size()) ? L[a.role_data] / 12 : 0;
        max_pts = std::max(max_pts, nd);
        for (size_t f = 0; f < L.size() && f < max_len.size(); ++f) {
          max_len[f] = std::max(max_len[f], L[f]);
          const uint64_t e = nd ? (L[f] + nd - 1) / nd : L[f];
          ext_elem[f] = std::max<uint32_t>(ext_elem[f], (uint32_t)std::max<uint64_t>(1, e));
        }
      }
    uint64_t cap = std::max<uint64_t>(max_pts, max_target);
    for (size_t f = 0; f < bytes_fields.size(); ++f) {
      if (!((tracked >> f) & 1u)) continue;
      uint32_t e = 1;
      if ((int)f == a.role_data || (int)f == a.role_normal || (int)f == a.role_color) e = 12;
      else if ((int)f == a.role_intensity) e = 4;
      else e = ext_elem[f];
      a.field_cap[f] = e;
      cap = std::max<uint64_t>(cap, (max_len[f] + e - 1) / e);
    }
    cap = std::max<uint64_t>(cap, 1);
    if (cap > (1u << 30)) fail(kOutOfBounds, "cloud too large");
    a.cap_points = (uint32_t)cap;
    a.max_blob = (uint32_t)max_blob;
    // static size analysis per tracked field: 0 = input size, 1 = fixed T,
    // 2 = data dependent (crop / voxel)
    std::vector<int> state(bytes_fields.size(), 0);
    std::vector<uint64_t> fixed_pts(bytes_fields.size(), 0);
    for (size_t k = 0; k < g.maps.size(); ++k) {
      const OpDesc& op = a.ops[k];
      uint32_t moved = 0;
      for (int r : {a.role_data, a.role_normal, a.role_color})
        if (r >= 0) moved |= 1u << r;
      if (op.kind == kFps || op.kind == kRangeCrop || op.kind == kVoxel || op.kind == kRandomCrop)
        if (a.role_intensity >= 0) moved |= 1u << a.role_intensity;
      moved |= op.gather_mask;
      if (op.kind == kVoxel) moved = tracked;
      for (size_t f = 0; f < bytes_fields.size(); ++f) {
        if (!((moved >> f) & 1u)) continue;
        if (op.kind == kDownsample || op.kind == kFps) {
          state[f] = 1;
          fixed_pts[f] = (uint64_t)op.num_points;
        } else if (op.kind == kRandomCrop || op.kind == kRangeCrop || op.kind == kVoxel) {
          state[f] = 2;
        }
      }
    }
    bool any_voxel = false, any_counts = false;
    for (int k = 0; k < a.n_ops; ++k)
      if (a.ops[k].kind == kVoxel) {
        any_voxel = true;
        any_counts |= a.ops[k].counts != 0;
      }
    a.voxel_scratch = any_voxel ? 1 : 0;
    a.count_out = -1;
    // outputs in std::map (name) order
    std::vector<int32_t> order(h.schema.size());
    for (size_t f = 0; f < order.size(); ++f) order[f] = (int32_t)f;
    std::sort(order.begin(), order.end(),
              [&](int32_t x, int32_t y) { return h.schema[x].name < h.schema[y].name; });
    for (int k = 0; k < kMaxBytesFields; ++k) a.bytes_out[k] = -1;
    for (int32_t f : order) {
      OutField o;
      o.name = h.schema[f].name;
      o.kind = h.schema[f].kind;
      o.schema_idx = f;
      const int bi = a.fields[f].bytes_index;
      if (bi >= 0) {
        if ((tracked >> bi) & 1u) {
          const uint64_t e = a.field_cap[bi];
          if (state[bi] == 1) o.stride = align4(fixed_pts[bi] * e);
          else if (state[bi] == 2) o.stride = align4(cap * e);
          else o.stride = align4(std::max<uint64_t>(max_len[bi], 1));
        } else {
          o.stride = align4(max_len[bi]);
        }
        a.bytes_out[bi] = (int32_t)outs.size();
      } else if (h.schema[f].kind == kString) {
        o.stride = 4096;
      } else {
        const uint64_t es = (h.schema[f].kind == kInt64 || h.schema[f].kind == kFloat64) ? 8 : 4;
        o.stride = es * h.schema[f].elems();
      }
      o.stride = std::max<uint64_t>(o.stride, 4);
      o.varlen = h.schema[f].kind == kBytes || h.schema[f].kind == kString;
      a.fields[f].out_index = (int32_t)outs.size();
      outs.push_back(o);
    }
    if (any_counts) {  // synthesized "count" bytes field (int32 per voxel)
      for (const auto& o : outs)
        if (o.name == "count") fail(kSchemaConflict, "schema already has a 'count' field");
      OutField o;
      o.name = "count";
      o.kind = kBytes;
      o.schema_idx = -1;
      o.stride = align4(cap * 4);
      o.varlen = true;
      size_t pos = 0;
      while (pos < outs.size() && outs[pos].name < o.name) ++pos;
      outs.insert(outs.begin() + pos, o);
      for (int f = 0; f < a.n_fields; ++f)
        if (a.fields[f].out_index >= (int32_t)pos) ++a.fields[f].out_index;
      for (int k = 0; k < kMaxBytesFields; ++k)
        if (a.bytes_out[k] >= (int32_t)pos) ++a.bytes_out[k];
      a.count_out = (int32_t)pos;
    }
    if (outs.size() > (size_t)PCP_MAX_BATCH_FIELDS) fail(kOutOfBounds, "too many batch fields");
    a.n_out = (int32_t)outs.size();
    var_index.assign(outs.size(), -1);
    n_var = 0;
    for (size_t f = 0; f < outs.size(); ++f)
      if (outs[f].varlen) var_index[f] = (int32_t)n_var++;
    // per-CTA buffer plan for k_cloud (sizes from the op chain, shared
    // memory by priority, the rest in a per-CTA global slab)
    bool any_stored_raw = false;
    for (const auto& bh : block_head) any_stored_raw |= !(bh.flags & kFlagOuterLz4);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    const size_t fixed = cloud_smem_fixed();
    plan_fps_cluster(a, (uint32_t)threads);
    a.op_begin = 0;
    a.op_end = a.n_ops;
    a.split_at = 0;
    a.vx_first = a.vx_last = -1;
    if (a.fps_cluster > 1) {  // run the ops before the first FPS one CTA per cloud
      int f = 0;
      while (f < a.n_ops && a.ops[f].kind != kFps) ++f;
      if (f > 0 && f < a.n_ops) a.split_at = f;
    }
    plan_vx(a);
    if (a.split_at || vx_on) {  // hand-off slot layout (fields sized like the per-CTA buffers)
      uint64_t at = 128;  // header: status, present, n[8], elem[8], has_counts, n_counts
      for (int k = 0; k < kMaxBytesFields; ++k) {
        a.handoff_off[k] = at;
        if ((a.tracked_mask >> k) & 1u) at = align16(at + (uint64_t)a.cap_points * a.field_cap[k] + 16);
      }
      a.handoff_off[kMaxBytesFields] = at;
      if (a.voxel_scratch) at = align16(at + 4ull * a.cap_points + 16);
      a.handoff_stride = at;
    }
    if (op_timing) {
      d_op_cycles.ensure((kMaxOps + 2) * 8);
      CK(cudaMemset(d_op_cycles.p, 0, (kMaxOps + 2) * 8));
      a.op_cycles = d_op_cycles.as<unsigned long long>();
    }
    const size_t used = plan_buffers(a, any_stored_raw, prop.sharedMemPerBlockOptin - fixed);
    smem = fixed + used;
    CK(set_cloud_smem(smem));
    // two CTAs per SM when the shared footprint allows it (the 64-register
    // build), otherwise (or with FPS: register-resident points) one CTA with
    // the 128-register build
    bool any_fps = false;
    for (int k = 0; k < a.n_ops; ++k) any_fps |= a.ops[k].kind == kFps;
    a.min_blocks = (2 * smem <= prop.sharedMemPerMultiprocessor && !any_fps) ? 2 : 1;
    if (a.fps_cluster > 1) {  // one cloud per cluster of fps_cluster CTAs
      int clusters = 0;
      CK(occupancy_cloud_clusters(&clusters, threads, smem, a.fps_cluster, false));
      if (clusters < 1) fail(kOutOfBounds, "no room for a cluster of " + std::to_string(a.fps_cluster) + " CTAs");
      grid = clusters * (int)a.fps_cluster;
      int per_sm = 0;  // the split's prefix launch: one CTA per cloud
      CK(occupancy_cloud(&per_sm, threads, smem, 1));
      grid_pre = std::max(1, per_sm) * sms;
    } else {
      int per_sm = 0;
      CK(occupancy_cloud(&per_sm, threads, smem, a.min_blocks));
      grid = std::max(1, per_sm) * sms;
    }
    a.force_serial_fy = force_serial_fy ? 1 : 0;
  }

  // The multi-CTA voxel stage takes the chain's leading [range_crop,] voxel
  // when clouds are large and the ops move exactly the tracked fields (so the
  // voxelized hand-off holds the whole cloud).
  void plan_vx(WaveArgs& a) {
    vx_on = false;
    if (!vx_allowed || a.n_ops == 0 || a.role_data < 0 || a.cap_points < vx_min_points) return;
    int first = 0, last = -1;
    if (a.ops[0].kind == kVoxel) last = 0;
    else if (a.ops[0].kind == kRangeCrop && a.n_ops > 1 && a.ops[1].kind == kVoxel) last = 1;
    if (last < 0) return;
    if (a.split_at && a.split_at <= last) return;
    const OpDesc& vo = a.ops[last];
    uint32_t mm = vo.gather_mask;
    for (int r : {a.role_data, a.role_normal, a.role_color, a.role_intensity})
      if (r >= 0) mm |= 1u << r;
    if (mm != a.tracked_mask) return;
    if (last == 1 && a.ops[0].gather_mask != vo.gather_mask) return;
    vx_on = true;
    a.vx_first = first;
    a.vx_last = last;
    VxArgs& v = vx_proto;
    std::memset(&v, 0, sizeof(v));
    v.n_bytes_fields = a.n_bytes_fields;
    v.role_data = a.role_data;
    v.role_normal = a.role_normal;
    v.role_color = a.role_color;
    v.role_intensity = a.role_intensity;
    v.mm = mm;
    v.has_crop = last == 1;
    for (int k = 0; k < 3; ++k) {
      v.lo[k] = a.ops[0].lo[k];
      v.hi[k] = a.ops[0].hi[k];
      v.origin[k] = vo.origin[k];
    }
    v.voxel = vo.voxel;
    v.has_origin = vo.has_origin;
    v.counts = vo.counts;
    v.vx_first = first;
    v.vx_last = last;
    v.max_passes = kVxMaxPasses;
    // bucket bits: ~1-2 points per bucket on average (dense surfaces still
    // split into shared-memory items), <= 20 bits
    const uint32_t cap_bits = 32u - (uint32_t)__builtin_clz(std::max<uint32_t>(a.cap_points, 2) - 1);
    v.bucket_bits = std::min<uint32_t>(kVxMaxBucketBits, cap_bits);
    v.bstride = 1u << v.bucket_bits;
    uint32_t pw = 0;
    for (int f = 0; f < a.n_bytes_fields; ++f)
      if ((mm >> f) & 1u) pw += (a.field_cap[f] + 3) / 4;
    v.pay_words = pw <= kVxMaxPayWords ? pw : 0;
  }


  void plan_waves() {
    const uint64_t n = walk.size();
    const uint32_t B = g.batch_size;
    uint32_t wb = wave_batches;
    if (!wb) {
      // default: >= 8192 samples and >= 2 pages (groups) per SM per wave, so
      // with two waves in flight every decoder slot (4 per SM) holds a page
      // whose serial LZ4 chain runs concurrently
      uint64_t gmax = 1;
      for (const auto& gr : h.groups) gmax = std::max<uint64_t>(gmax, gr.sample_count);
      uint64_t want = std::max<uint64_t>(8192, 2ull * sms * gmax);
      // multi-CTA voxel chains: ~64 M input points per wave, so the per-wave
      // hand-off slots and sort words of several waves in flight stay modest
      if (vx_on) want = std::max<uint64_t>(B, (64ull << 20) / std::max<uint64_t>(1, proto.cap_points));
      wb = (uint32_t)std::max<uint64_t>(1, (want + B - 1) / B);
    }
    const uint64_t W = (uint64_t)wb * B;
    cur_wave_batches = wb;
    const uint64_t usable = g.drop_remainder ? (n / B) * B : n;
    // (re)plan from the end of the waves already launched (live
    // reconfiguration keeps the walk, the seeds and the batch boundaries)
    uint64_t e0 = 0, p0 = 0;
    if (next_plan > 0) {
      e0 = plan[next_plan - 1].first;
      p0 = plan[next_plan - 1].second + plan_n[next_plan - 1];
      if (p0 >= usable) ++e0, p0 = 0;
    }
    plan.resize(next_plan);
    plan_n.resize(next_plan);
    for (uint64_t e = e0; e < epochs; ++e)
      for (uint64_t p = e == e0 ? p0 : 0; p < usable; p += W) {
        plan.push_back({e, p});
        plan_n.push_back(std::min<uint64_t>(W, usable - p));
      }
  }

  // Groups a wave touches, in first-use order (the wave's page order).
  std::vector<uint32_t> wave_groups(uint64_t pos0, uint64_t n) const {
    std::vector<uint32_t> groups;
    std::vector<char> seen(h.groups.size(), 0);
    for (uint64_t k = 0; k < n; ++k) {
      const uint32_t gi = walk[pos0 + k].group_index;
      if (!seen[gi]) {
        seen[gi] = 1;
        groups.push_back(gi);
      }
    }
    return groups;
  }

  // Where a wave's pages sit: resident -> their byte-store offsets; staged ->
  // a device staging buffer.  A wave's pages are consecutive groups of a few
  // slices, so their byte ranges are sorted and merged (gaps <= 64 KiB copied
  // along): a handful of large H2D copies (and file reads) per wave instead of
  // two per group.  stage_off[kind * ng + i] = page offset; runs = (store
  // offset, length) copied to [64, stage_at) with 64 B between runs.
  void stage_plan(const std::vector<uint32_t>& groups, std::vector<std::pair<uint64_t, uint64_t>>& runs,
                  std::vector<uint64_t>& stage_off, uint64_t& stage_at) const {
    const uint32_t ng = (uint32_t)groups.size();
    stage_off.assign(2 * ng, 0);
    runs.clear();
    stage_at = 64;
    struct PRun {
      uint64_t lo, hi;
      uint32_t page;
    };
    std::vector<PRun> prs;
    for (uint32_t i = 0; i < ng; ++i) {
      const Group& gr = h.groups[groups[i]];
      for (int kind = 0; kind < 2; ++kind) {
        const uint64_t so = slice_base[gr.slice] + (kind ? gr.block_off : gr.scalar_off);
        const uint64_t len = kind ? gr.block_len : gr.scalar_len;
        if (!resident) prs.push_back({so, so + len, (uint32_t)(kind * ng + i)});
        else stage_off[kind * ng + i] = so;
      }
    }
    if (resident || prs.empty()) return;
    std::sort(prs.begin(), prs.end(), [](const PRun& x, const PRun& y) { return x.lo < y.lo; });
    size_t k = 0;
    while (k < prs.size()) {
      const uint64_t lo = prs[k].lo & ~uint64_t(15);
      uint64_t hi = align16(prs[k].hi);
      size_t e = k + 1;
      while (e < prs.size() && prs[e].lo <= hi + 65536) hi = std::max(hi, align16(prs[e].hi)), ++e;
      for (size_t q = k; q < e; ++q) stage_off[prs[q].page] = stage_at + (prs[q].lo - lo);
      runs.push_back({lo, hi - lo});
      stage_at += (hi - lo) + 64;
      k = e;
    }
  }

  // ---- file streaming: reader threads fill slot (pi % slots) with wave pi --
  void reader_main() {
    try {
      CK(cudaSetDevice(device));
      const size_t ns = slots.size();
      for (size_t pi = 0; pi < plan.size(); ++pi) {
        const size_t si = pi % ns;
        {
          std::unique_lock<std::mutex> lk(rd_mu);
          // the slot's previous wave must have been launched (its copies enqueued)
          rd_cv.wait(lk, [&] { return rd_stop || pi < ns || launched_upto >= (int64_t)(pi - ns); });
          if (rd_stop) return;
        }
        Wave& w = slots[si];
        if (pi >= ns) CK(cudaEventSynchronize(w.h1));  // its H2D copies out of h_stage are done
        std::vector<std::pair<uint64_t, uint64_t>> runs;
        std::vector<uint64_t> stage_off;
        uint64_t stage_at = 64;
        stage_plan(wave_groups(plan[pi].second, plan_n[pi]), runs, stage_off, stage_at);
        w.h_stage.ensure(stage_at + 64);
        // chunks of <= 4 MiB over the reader threads
        std::vector<std::array<uint64_t, 3>> chunks;  // store lo, len, h_stage offset
        uint64_t d_at = 64;
        for (const auto& r : runs) {
          for (uint64_t o = 0; o < r.second; o += (4ull << 20))
            chunks.push_back({r.first + o, std::min<uint64_t>(4ull << 20, r.second - o), d_at + o});
          d_at += r.second + 64;
        }
        std::atomic<size_t> next{0};
        std::string err;
        std::mutex err_mu;
        auto work = [&] {
          for (size_t c; (c = next.fetch_add(1)) < chunks.size();) {
            try {
              read_store_range(chunks[c][0], chunks[c][1], w.h_stage.as<uint8_t>() + chunks[c][2]);
            } catch (const std::exception& e) {
              std::lock_guard<std::mutex> l(err_mu);
              err = e.what();
            }
          }
        };
        std::vector<std::thread> pool;
        const size_t nt = std::min<size_t>(reader_threads, chunks.size());
        for (size_t t = 1; t < nt; ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
        if (!err.empty()) fail(kIoFailure, err);
        {
          std::lock_guard<std::mutex> lk(rd_mu);
          ready_upto = (int64_t)pi;
          read_bytes += d_at;
        }
        rd_cv.notify_all();
      }
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lk(rd_mu);
      rd_err = e.what();
      rd_failed = true;
      rd_cv.notify_all();
    }
  }

  // ---- wave construction ---------------------------------------------------
  void launch(Wave& w, size_t pi, bool dry = false) {
    // the slot's previous wave may still be read by copies the user enqueued
    // on the serve stream (pcp_memcpy_d2h_async): overwrite after them
    if (!dry && w.served) CK(cudaStreamWaitEvent(w.stream, w.served, 0));
    w.epoch = plan[pi].first;
    w.pos0 = plan[pi].second;
    w.n = plan_n[pi];
    const uint32_t B = g.batch_size;
    w.first_batch = w.pos0 / B;
    w.n_batches = (uint32_t)((w.n + B - 1) / B);
    WaveArgs a = proto;
    // groups touched, in first-use order
    std::map<uint32_t, uint32_t> gmap;  // header group index -> wave group
    std::vector<uint32_t> groups;
    std::vector<uint32_t> rows_seen;  // per wave group: bitmap count check
    std::vector<std::vector<uint32_t>> hits;
    for (uint64_t k = 0; k < w.n; ++k) {
      const Entry& e = walk[w.pos0 + k];
      auto it = gmap.find(e.group_index);
      if (it == gmap.end()) {
        gmap.emplace(e.group_index, (uint32_t)groups.size());
        groups.push_back(e.group_index);
        hits.emplace_back(h.groups[e.group_index].sample_count, 0);
      }
      hits[gmap[e.group_index]][e.row]++;
    }
    const uint32_t ng = (uint32_t)groups.size();
    // pages: [0, ng) scalar, [ng, 2ng) block
    std::vector<PageRef> pages(2 * ng);
    std::vector<GroupWork> gw(ng);
    std::vector<uint32_t> todo;
    std::vector<uint64_t> todo_scratch;
    uint64_t scratch_at = 0;
    auto add_todo = [&](uint32_t page, const PageHead& ph) {
      todo.push_back(page);
      todo_scratch.push_back(scratch_at);
      if (ph.flags & kFlagOuterLz4) scratch_at = align16(scratch_at + lz4_scratch_bytes(ph.pay_len));
    };
    std::vector<CrcWindow> wins;
    uint64_t raw_at = 0, vals_at = 0;
    uint32_t rec_at = 0;
    std::vector<std::pair<uint64_t, uint64_t>> runs;  // (store off, len), 16-B aligned
    uint64_t stage_at = 64;
    std::vector<uint64_t> stage_off;
    stage_plan(groups, runs, stage_off, stage_at);
    for (uint32_t i = 0; i < ng; ++i) {
      const uint32_t gi = groups[i];
      const Group& gr = h.groups[gi];
      const PageHead& sh = scalar_head[gi];
      const PageHead& bh = block_head[gi];
      PageRef& sp = pages[i];
      sp.off = stage_off[i];
      sp.raw_len = sh.raw_len;
      sp.pay_len = sh.pay_len;
      sp.crc = sh.crc;
      sp.flags = sh.flags;
      sp.raw_dst = raw_at;
      raw_at = align16(raw_at + sh.raw_len) + 16;
      sp.crc_mode = 0;
      add_todo(i, sh);
      PageRef& bp = pages[ng + i];
      bp.off = stage_off[ng + i];
      bp.raw_len = bh.raw_len;
      bp.pay_len = bh.pay_len;
      bp.crc = bh.crc;
      bp.flags = bh.flags;
      bp.raw_dst = ~uint64_t(0);
      if (bh.flags & kFlagOuterLz4) {
        bp.raw_dst = raw_at;
        raw_at = align16(raw_at + bh.raw_len) + 16;
        add_todo(ng + i, bh);
      }
      // fused CRC only when this wave's samples tile the stored-raw payload
      // exactly once
      // (not with the vx stage: one CTA would CRC a whole multi-MB blob; the
      // windowed kernel spreads it over the GPU)
      bool fused = !(bh.flags & kFlagOuterLz4) && bh.pay_len == bh.raw_len && !no_fused_crc && !vx_on;
      uint64_t at = 0;
      for (uint32_t r = 0; fused && r < gr.sample_count; ++r) {
        if (hits[i][r] != 1 || gr.blob_ranges[r][0] != at) fused = false;
        at = gr.blob_ranges[r][1];
      }
      if (at != bh.raw_len) fused = false;
      bp.crc_mode = fused ? 1 : 0;
      for (uint32_t kind = 0; kind < 2; ++kind) {
        const PageRef& p = pages[kind * ng + i];
        if (kind == 1 && p.crc_mode == 1) continue;
        const uint64_t pay0 = p.off + kPageHeaderBytes;
        const uint64_t win = 65536;
        for (uint64_t end = p.pay_len; end > 0;) {
          const uint64_t st = end > win ? end - win : 0;
          wins.push_back({pay0 + st, end - st, p.pay_len - end, kind * ng + i, 0});
          end = st;
        }
      }
      gw[i].scalar_page = i;
      gw[i].first_rec = rec_at;
      gw[i].n_rows = gr.sample_count;
      gw[i].vals_base = (uint32_t)vals_at;
      rec_at += gr.sample_count;
      // value bytes per row: fixed fields + strings (bounded by the page)
      uint64_t fixed = 0;
      bool has_string = false;
      for (const auto& f : h.schema) {
        if (f.kind == kBytes) continue;
        if (f.kind == kString) { has_string = true; fixed += 4; continue; }
        fixed += ((f.kind == kInt64 || f.kind == kFloat64) ? 8 : 4) * (uint64_t)f.elems();
      }
      vals_at += fixed * gr.sample_count + (has_string ? sh.raw_len : 0);
      vals_at = align16(vals_at);
    }
    std::vector<SampleWork> sw(w.n);
    w.in_payload_bytes = 0;
    w.in_points = 0;
    for (uint64_t k = 0; k < w.n; ++k) {
      const Entry& e = walk[w.pos0 + k];
      SampleWork& s = sw[k];
      s.epoch = w.epoch;
      s.index = w.pos0 + k;
      s.blob_start = e.blob_start;
      s.blob_end = e.blob_end;
      s.group = gmap[e.group_index];
      s.scalar_page = s.group;
      s.block_page = ng + s.group;
      s.row = e.row;
      w.in_payload_bytes += e.blob_end - e.blob_start;
      const auto& L = h.groups[e.group_index].blob_lens[e.row];
      if (a.role_data >= 0 && a.role_data < (int)L.size()) w.in_points += L[a.role_data] / 12;
    }
    // ---- pack tables into one pinned blob, one H2D copy ---------------------
    auto sz = [](uint64_t v) { return align16(v); };
    const uint64_t o_pages = 0;
    const uint64_t o_groups = o_pages + sz(pages.size() * sizeof(PageRef));
    const uint64_t o_samples = o_groups + sz(gw.size() * sizeof(GroupWork));
    const uint64_t o_todo = o_samples + sz(sw.size() * sizeof(SampleWork));
    const uint64_t o_tsc = o_todo + sz(todo.size() * 4);
    const uint64_t o_wins = o_tsc + sz(todo.size() * 8);
    const uint64_t up_bytes = o_wins + sz(wins.size() * sizeof(CrcWindow));
    // device-only regions after the uploaded part
    const uint64_t o_recs = up_bytes;
    const uint64_t o_vals = o_recs + sz((uint64_t)rec_at * sizeof(ScalarRec));
    const uint64_t o_acc = o_vals + sz(vals_at + 16);
    const uint64_t o_pst = o_acc + sz(pages.size() * 4);
    const uint64_t o_sst = o_pst + sz(pages.size() * 4);
    const uint64_t o_sop = o_sst + sz(w.n * 4);
    const uint64_t o_swh = o_sop + sz(w.n * 4);
    const uint64_t o_len = o_swh + sz(w.n * 4);
    const uint64_t o_woff = o_len + sz(outs.size() * w.n * 8);
    const uint64_t o_dense = o_woff + sz((uint64_t)n_var * (w.n + 1) * 8);
    const uint64_t total = o_dense + sz(outs.size() * 4);
    // size every buffer first (a dry run stops here: open() pre-sizes the
    // slots for the largest planned wave so no cudaMalloc lands mid-run)
    w.h_tables.ensure(up_bytes);
    w.tables.ensure(total);
    if (!resident) w.bytes_stage.ensure(stage_at + 64);
    w.raw.ensure(raw_at + 64);
    w.lz4_scratch.ensure(scratch_at + 64);
    w.out_base.resize(outs.size());
    uint64_t out_total = 0;
    for (size_t f = 0; f < outs.size(); ++f) {
      w.out_base[f] = out_total;
      out_total += align16(outs[f].stride * w.n) + 64;
    }
    w.outs.ensure(out_total);
    if (n_var) w.compact.ensure(out_total);
    // host_batches: size the pinned wave buffer up front (exact for fixed-size
    // fields; ragged ones grow it on demand past 1 GiB)
    if (host_batches) w.h_out.ensure(std::min<uint64_t>(out_total + 64, 1ull << 30));
    if (proto.split_at || vx_on) w.handoff.ensure(proto.handoff_stride * w.n);
    uint64_t vx_tiles_bound = 0, vx_btiles_bound = 0, vx_max_items = 0;
    if (vx_on) {
      const uint64_t T = voxel_wave_tile_points();
      vx_tiles_bound = w.n * ((proto.cap_points + T - 1) / T);
      vx_btiles_bound = w.n * ((proto.cap_points + kVxBTile - 1) / kVxBTile);
      vx_max_items = proto.cap_points / (kVxItemCap / 2) + 2;
      w.vx_bt.ensure(16 + 4 * vx_btiles_bound);
      w.vx_bcnt.ensure(4ull * vx_proto.bstride * w.n);
      w.vx_boff.ensure(4ull * (vx_proto.bstride + 4) * w.n);  // per-cloud rows 16-B aligned
      w.vx_items.ensure(8ull * vx_max_items * w.n);
      w.vx_T.ensure(proto.handoff_stride * w.n);
      w.handoff_b.ensure(proto.handoff_stride * w.n);
      w.vx_cl.ensure(sizeof(VxCloud) * w.n);
      w.vx_tiles.ensure(16 + 3 * 4 * vx_tiles_bound);
      w.vx_cnt.ensure(1024 * vx_tiles_bound);
      w.vx_w0.ensure(8ull * proto.cap_points * w.n);
      w.vx_w1.ensure(3 * 8ull * proto.cap_points * w.n);  // LSD pong + bucket-mode dense-item buffers
    }
    if (proto.n_rng) w.mt_pre.ensure(w.n * proto.n_rng * 312 * 8);
    w.h_res.ensure(total - o_sst + 16);
    // phase 4 of the LZ4 pages: page-wide pointer jumping, or a warp per page
    // for pages of many small clouds (C2's 64 x 32 KB: float literals the warp
    // skips and short label chains), where it measured faster
    uint32_t n_lz4 = 0, max_raw = 0;
    uint64_t lz4_block_samples = 0, n_lz4_block = 0;
    for (uint32_t pg_i : todo)
      if (pages[pg_i].flags & kFlagOuterLz4) {
        ++n_lz4;
        max_raw = std::max<uint32_t>(max_raw, (uint32_t)std::min<uint64_t>(pages[pg_i].raw_len, 0xFFFFFFFFull));
        if (pg_i >= ng) {
          ++n_lz4_block;
          lz4_block_samples += h.groups[groups[pg_i - ng]].sample_count;
        }
      }
    // (waves whose only LZ4 pages are the small scalar pages keep the warp:
    // a pages x 64 grid of near-empty CTAs per round would only crowd the SMs)
    const bool many_small = n_lz4_block > 0 && lz4_block_samples >= 32 * n_lz4_block;
    const bool pj = n_lz4 > 0 && (lz4_pj > 0 || (lz4_pj < 0 && n_lz4_block > 0 && !many_small));
    uint32_t pj_rounds = 0;
    if (pj) {
      pj_rounds = (max_raw > 1 ? 32u - __builtin_clz(max_raw - 1) : 0u) + 1u;  // ceil(log2) + 1
      w.pj_ptr.ensure(4ull * (raw_at + 64));
      w.pj_changed.ensure(4ull * pj_rounds * todo.size() + 64);
      w.pj_flags.ensure(raw_at / 256 + todo.size() + 64);  // per 256-B block (+1 per page)
    }
    if (dry) return;
    if (pj) ++lz4_pj_waves;
    uint8_t* ht = w.h_tables.as<uint8_t>();
    std::memcpy(ht + o_pages, pages.data(), pages.size() * sizeof(PageRef));
    std::memcpy(ht + o_groups, gw.data(), gw.size() * sizeof(GroupWork));
    std::memcpy(ht + o_samples, sw.data(), sw.size() * sizeof(SampleWork));
    std::memcpy(ht + o_todo, todo.data(), todo.size() * 4);
    std::memcpy(ht + o_tsc, todo_scratch.data(), todo_scratch.size() * 8);
    std::memcpy(ht + o_wins, wins.data(), wins.size() * sizeof(CrcWindow));
    uint8_t* dt = w.tables.as<uint8_t>();
    // staged input bytes
    const uint8_t* bytes = d_store.as<uint8_t>();
    CK(cudaEventRecord(w.h0, w.stream));
    if (!resident && stream_files) {
      // the reader threads filled this slot's pinned buffer with the wave's
      // runs (same layout as bytes_stage): one H2D copy
      const auto t0 = std::chrono::steady_clock::now();
      {
        std::unique_lock<std::mutex> lk(rd_mu);
        rd_cv.wait(lk, [&] { return rd_failed || ready_upto >= (int64_t)pi; });
        if (rd_failed) fail(kIoFailure, "slice read: " + rd_err);
      }
      read_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      CK(cudaMemcpyAsync(w.bytes_stage.as<uint8_t>() + 64, w.h_stage.as<uint8_t>() + 64, stage_at - 64,
                         cudaMemcpyHostToDevice, w.stream));
      bytes = w.bytes_stage.as<uint8_t>();
      for (const auto& r : runs) h2d_bytes += r.second;
    } else if (!resident) {
      uint64_t d_at = 64;
      for (const auto& r : runs) {
        CK(cudaMemcpyAsync(w.bytes_stage.as<uint8_t>() + d_at, h_store.as<uint8_t>() + r.first,
                           r.second, cudaMemcpyHostToDevice, w.stream));
        d_at += r.second + 64;
      }
      bytes = w.bytes_stage.as<uint8_t>();
      for (const auto& r : runs) h2d_bytes += r.second;
    }
    CK(cudaMemcpyAsync(dt, ht, up_bytes, cudaMemcpyHostToDevice, w.stream));
    CK(cudaEventRecord(w.h1, w.stream));
    if (stream_files) {  // the reader may refill this slot's buffer once h1 completes
      {
        std::lock_guard<std::mutex> lk(rd_mu);
        launched_upto = (int64_t)pi;
      }
      rd_cv.notify_all();
    }
    CK(cudaMemsetAsync(dt + o_acc, 0, o_woff - o_acc, w.stream));  // incl. out_len: failed samples write none
    // ---- args ----------------------------------------------------------------
    a.bytes = bytes;
    a.raw = w.raw.as<uint8_t>();
    a.pages = reinterpret_cast<const PageRef*>(dt + o_pages);
    a.n_pages = (uint32_t)pages.size();
    a.groups = reinterpret_cast<const GroupWork*>(dt + o_groups);
    a.n_groups = ng;
    a.samples = reinterpret_cast<const SampleWork*>(dt + o_samples);
    a.n_samples = (uint32_t)w.n;
    a.recs = reinterpret_cast<ScalarRec*>(dt + o_recs);
    a.vals = dt + o_vals;
    a.page_crc_acc = reinterpret_cast<uint32_t*>(dt + o_acc);
    a.page_status = reinterpret_cast<int32_t*>(dt + o_pst);
    a.sample_status = reinterpret_cast<int32_t*>(dt + o_sst);
    a.sample_op = reinterpret_cast<int32_t*>(dt + o_sop);
    a.sample_where = reinterpret_cast<int32_t*>(dt + o_swh);
    a.out_len = reinterpret_cast<uint64_t*>(dt + o_len);
    a.shift_tab = d_shift.as<uint32_t>();
    a.gscratch = proto.gscratch_per_cta ? w.gscratch.as<uint8_t>() : nullptr;
    a.handoff_in = a.handoff_out = a.handoff_fallback = nullptr;
    a.vx_state = nullptr;
    VxArgs vx = vx_proto;
    if (vx_on) {
      vx.n_samples = (uint32_t)w.n;
      vx.A = w.handoff.as<uint8_t>();
      vx.B = w.handoff_b.as<uint8_t>();
      vx.stride = proto.handoff_stride;
      for (int k = 0; k <= kMaxBytesFields; ++k) vx.off[k] = proto.handoff_off[k];
      vx.cl = w.vx_cl.as<VxCloud>();
      vx.total_tiles = w.vx_tiles.as<uint32_t>();
      vx.tile_cloud = vx.total_tiles + 4;
      vx.tile_kept = vx.tile_cloud + vx_tiles_bound;
      vx.tile_kofs = vx.tile_kept + vx_tiles_bound;
      vx.cnt = w.vx_cnt.as<uint32_t>();
      vx.w0 = w.vx_w0.as<uint64_t>();
      vx.w1 = w.vx_w1.as<uint64_t>();
      vx.w2 = vx.w1 + (uint64_t)proto.cap_points * w.n;
      vx.total_btiles = w.vx_bt.as<uint32_t>();
      vx.btile_cloud = vx.total_btiles + 4;
      vx.bcur = w.vx_bcnt.as<uint32_t>();
      vx.any_lsd = vx.total_btiles + 1;
      vx.boff = w.vx_boff.as<uint32_t>();
      vx.item_v = w.vx_items.as<uint32_t>();
      vx.item_b = vx.item_v + vx_max_items * w.n;
      vx.max_items = (uint32_t)vx_max_items;
      vx.T = w.vx_T.as<uint8_t>();
      vx.msd_enabled = vx_msd ? 1 : 0;
      vx.sample_status = a.sample_status;
      vx.sample_op = a.sample_op;
      vx.sample_where = a.sample_where;
      a.vx_state = vx.cl;
      a.handoff_fallback = vx.A;
    }
    a.mt_pre = proto.n_rng ? w.mt_pre.as<uint64_t>() : nullptr;
    for (size_t f = 0; f < outs.size(); ++f) {
      a.out[f] = w.outs.as<uint8_t>() + w.out_base[f];
      a.out_stride[f] = outs[f].stride;
    }
    // ---- kernels ---------------------------------------------------------------
    CK(cudaEventRecord(w.c0, w.stream));
    CK(launch_crc_windows(bytes, reinterpret_cast<const CrcWindow*>(dt + o_wins),
                          (uint32_t)wins.size(), d_shift.as<uint32_t>(), a.page_crc_acc, sms, w.stream));
    CK(cudaEventRecord(w.c1, w.stream));
    w.crc_alg_bytes = 0;
    for (const auto& cw : wins) w.crc_alg_bytes += cw.len;
    long long* tm = nullptr;
    if (lz4_timing) {  // PCP_LZ4_TIMING=1: per-page phase clocks (diagnostics)
      w.lz4_timing.ensure(todo.size() * 128);
      CK(cudaMemsetAsync(w.lz4_timing.p, 0, todo.size() * 128, w.stream));
      tm = w.lz4_timing.as<long long>();
    }
    CK(cudaEventRecord(w.d0, w.stream));
    CK(launch_page_decode(bytes, a.raw, a.pages, reinterpret_cast<const uint32_t*>(dt + o_todo),
                          reinterpret_cast<const uint64_t*>(dt + o_tsc), w.lz4_scratch.as<uint8_t>(),
                          (uint32_t)todo.size(), a.page_status, w.stream, tm,
                          pj ? w.pj_ptr.as<uint32_t>() : nullptr, pj ? w.pj_changed.as<uint32_t>() : nullptr,
                          pj_rounds, pj ? w.pj_flags.as<uint8_t>() : nullptr,
                          (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(64, ((uint64_t)max_raw + 65535) / 65536))));
    CK(cudaEventRecord(w.d1, w.stream));
    w.n_todo = (uint32_t)todo.size();
    w.decode_alg_bytes = 0;
    for (uint32_t pi : todo) w.decode_alg_bytes += pages[pi].pay_len + pages[pi].raw_len;
    // the pipeline's second wave starts its op chain after the first wave's:
    // launched together, the two waves split every SM between their clouds
    // and the pipeline could stay in a slow interleaved regime for a whole run
    // (S3DIS: ~57 instead of ~35 ms per wave in about a third of fresh 10-epoch
    // runs; tools/s3dis_var3.py); with the first wave leading, later waves
    // fill SMs as its clouds finish (6 of 6 runs 6.4-6.8 K rooms/s)
    if (stagger_start && waves_launched_total == 1 && first_k1) CK(cudaStreamWaitEvent(w.stream, first_k1, 0));
    CK(launch_wave(a, grid, grid_pre, threads, smem, w.stream, w.k0, w.k1, vx_on ? &vx : nullptr,
                   (uint32_t)vx_tiles_bound, (uint32_t)vx_btiles_bound, sms, w.v0, w.v1, w.handoff.as<uint8_t>()));
    if (waves_launched_total++ == 0) first_k1 = w.k1;
    launches += (wins.empty() ? 0 : 1) + (todo.empty() ? 0 : 2) + (ng ? 1 : 0) + (proto.n_rng ? 1 : 0) + 1 + 1 + 1 +
                (vx_on ? 2 + 14 + 3 * kVxMaxPasses : 0) + (proto.split_at ? 1 : 0);
    if (vx_on) {
      uint64_t per_pt = 0;
      for (int f = 0; f < proto.n_bytes_fields; ++f)
        if ((proto.tracked_mask >> f) & 1u) per_pt += proto.field_cap[f];
      w.vx_alg_bytes = w.in_points * per_pt;
    }
    // ---- per-wave CSR of the variable-length fields (device side) ------------
    {
      WaveCsr c{};
      c.n_out = (uint32_t)outs.size();
      c.n_var = n_var;
      for (size_t f = 0; f < outs.size(); ++f) {
        c.stride[f] = outs[f].stride;
        c.var_index[f] = var_index[f];
        if (var_index[f] >= 0) c.var_field[var_index[f]] = (int32_t)f;
        c.outs[f] = w.outs.as<uint8_t>() + w.out_base[f];
        c.compact[f] = n_var ? w.compact.as<uint8_t>() + w.out_base[f] : nullptr;
      }
      c.woff = reinterpret_cast<uint64_t*>(dt + o_woff);
      c.dense = reinterpret_cast<uint32_t*>(dt + o_dense);
      CK(cudaEventRecord(w.s0, w.stream));
      CK(launch_wave_csr(a.out_len, c, (uint32_t)w.n, sms, w.stream));
      CK(cudaEventRecord(w.s1, w.stream));
      launches += 1 + (n_var ? 1 : 0);
    }
    h2d_bytes += up_bytes;
    // ---- results back to pinned host -------------------------------------------

    uint8_t* hr = w.h_res.as<uint8_t>();
    w.h_status = reinterpret_cast<int32_t*>(hr);
    w.h_op = reinterpret_cast<int32_t*>(hr + align16(w.n * 4));
    w.h_where = reinterpret_cast<int32_t*>(hr + 2 * align16(w.n * 4));
    w.h_len = reinterpret_cast<uint64_t*>(hr + (o_len - o_sst));
    w.h_woff = reinterpret_cast<uint64_t*>(hr + (o_woff - o_sst));
    w.h_dense = reinterpret_cast<uint32_t*>(hr + (o_dense - o_sst));
    w.staged = 0;
    // one contiguous region: the host layout mirrors o_sst..total
    static_assert(sizeof(int32_t) == 4, "");
    uint8_t* hr_dev = nullptr;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hr_dev), hr, 0));
    CK(launch_store_host(dt + o_sst, hr_dev, total - o_sst, w.stream));
    ++launches;
    CK(cudaEventRecord(w.done, w.stream));
    w.launched = true;
  }

  std::string op_message(int32_t st, int32_t op, int32_t where) const {
    uint32_t node = g.source_id;
    if (op >= 1 && op <= (int32_t)g.maps.size()) node = g.maps[op - 1].node_id;
    std::string what;
    switch (st) {
      case kChecksumMismatch: what = "block page checksum"; break;
      case kCorruptPage: what = where ? "corrupt page (lz4 stream / stored length)" : "record truncated"; break;
      case kRangeOutOfBounds: what = "blob range outside block page"; break;
      case kMissingField: what = "sample has no usable coordinates / missing field"; break;
      case kEmptyCloud: what = "zero points"; break;
      case kOutOfBounds: what = "index or size out of bounds"; break;
      case kUnknownOp: what = "unknown map"; break;
      default: what = "device failure"; break;
    }
    return "op " + std::to_string(node) + ": " + errc_name(st) + ": " + what;
  }

  // host_batches: once a wave's kernels are done, its batch fields go to
  // pinned host memory on the serve stream: one D2H per field per wave (dense
  // fields from their contiguous slots, variable-length fields from the
  // wave's device CSR).  Only samples [0, lim) are copied: the batches before
  // a wave's first failing batch are served intact, the failing one raises.
  void stage_host(Wave& w, uint64_t lim) {
    w.h_base.assign(outs.size(), 0);
    uint64_t total = 0;
    std::vector<uint64_t> bytes(outs.size(), 0);
    for (size_t f = 0; f < outs.size(); ++f) {
      bytes[f] = field_offset(w, f, lim);
      w.h_base[f] = total;
      total = align16(total + bytes[f]) + 64;
    }
    w.h_out.ensure(total + 64);
    uint8_t* ho = w.h_out.as<uint8_t>();
    for (size_t f = 0; f < outs.size(); ++f) {
      if (bytes[f]) CK(cudaMemcpyAsync(ho + w.h_base[f], field_base(w, f), bytes[f], cudaMemcpyDeviceToHost,
                                       serve_stream));
      d2h_bytes += bytes[f];
    }
    CK(cudaEventRecord(w.host_ready, serve_stream));
    CK(cudaEventSynchronize(w.host_ready));
    w.staged = lim;
  }

  // Batch field layout of a finished wave: dense fields (every sample fills
  // its slot) are their slots; variable-length ones live in the wave's CSR.
  bool field_dense(const Wave& w, size_t f) const { return !outs[f].varlen || w.h_dense[f] != 0; }
  uint64_t field_offset(const Wave& w, size_t f, uint64_t s) const {
    return field_dense(w, f) ? s * outs[f].stride : w.h_woff[(uint64_t)var_index[f] * (w.n + 1) + s];
  }
  const uint8_t* field_base(const Wave& w, size_t f) const {
    return (field_dense(w, f) ? w.outs.as<uint8_t>() : w.compact.as<uint8_t>()) + w.out_base[f];
  }

  // ---- iteration -------------------------------------------------------------
  int next_batch(pcp_batch* out, int* eos) {
    *eos = 0;
    ++sink_polls;
    if (failed) fail(fail_code, fail_msg);
    if (cur < 0 || served >= slots[cur].n_batches) {
      const int ns = (int)slots.size();
      using clk = std::chrono::steady_clock;
      auto ms_since = [](clk::time_point t0) {
        return std::chrono::duration<double, std::milli>(clk::now() - t0).count();
      };
      if (cur >= 0) {
        // every batch of the served wave was handed out: its slot is free once
        // the copies the user enqueued on the serve stream are done (the next
        // wave in it waits on this event on the device)
        ++waves_done;
        CK(cudaEventRecord(slots[cur].served, serve_stream));
        slots[cur].launched = false;
      }
      int nxt = cur < 0 ? 0 : (cur + 1) % ns;
      if (has_pending && !slots[nxt].launched) {
        bool busy = false;
        for (const auto& w : slots) busy |= w.launched;
        if (!busy) {  // drained: apply (Pipeline::update_op_config, pipeline.cpp:691-732)
          apply_config();
          nxt = 0;
        }
      }
      Wave& wn = slots[nxt];
      if (!wn.launched) {
        if (next_plan >= plan.size()) {
          *eos = 1;
          cur = -1;  // repeated calls stay at end of stream
          return kOk;
        }
        const auto t0 = clk::now();
        launch(wn, next_plan++);
        host_launch_ms += ms_since(t0);
      }
      // keep every slot busy while waiting: waves go to slots in ring order
      // on per-slot streams, so up to `slots` waves overlap (copies, LZ4
      // chains and k_cloud of different waves).  "serial": one wave at a time.
      for (int d = 1; d < (int)slots.size() && next_plan < plan.size() && !serial && !has_pending; ++d) {
        Wave& wp = slots[(nxt + d) % slots.size()];
        if (!wp.launched) {
          const auto t0 = clk::now();
          launch(wp, next_plan++);
          host_launch_ms += ms_since(t0);
        }
      }
      const auto tw = clk::now();
      if (cudaEventQuery(wn.done) == cudaErrorNotReady) ++sink_empty_polls;  // the consumer waits on the device
      CK(cudaEventSynchronize(wn.done));
      host_wait_ms += ms_since(tw);
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, wn.k0, wn.k1));
      cloud_kernel_ms += ms;
      if (vx_on) {  // the vx stage runs between the k_cloud launches
        CK(cudaEventElapsedTime(&ms, wn.v0, wn.v1));
        cloud_kernel_ms -= ms;
        vx_kernel_ms += ms;
        vx_alg_bytes += wn.vx_alg_bytes;
      }
      CK(cudaEventElapsedTime(&ms, wn.d0, wn.d1));
      decode_kernel_ms += ms;
      CK(cudaEventElapsedTime(&ms, wn.c0, wn.c1));
      crc_kernel_ms += ms;
      crc_alg_bytes += wn.crc_alg_bytes;
      CK(cudaEventElapsedTime(&ms, wn.s0, wn.s1));
      csr_kernel_ms += ms;
      for (size_t f = 0; f < outs.size(); ++f)  // bytes moved by k_compact_wave (read + write)
        if (!field_dense(wn, f)) csr_alg_bytes += 2 * field_offset(wn, f, wn.n);
      if (timeline_on) {  // PCP_TIMELINE=1: per-wave event times (ms from open)
        std::vector<double> row;
        for (cudaEvent_t e : {wn.h0, wn.h1, wn.d0, wn.d1, wn.k0, wn.k1, wn.done}) {
          float t = 0;
          CK(cudaEventElapsedTime(&t, t_open, e));
          row.push_back(t);
        }
        row.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_open).count());
        timeline.push_back(row);
      }
      decode_alg_bytes += wn.decode_alg_bytes;
      if (lz4_timing && wn.n_todo) {
        std::vector<long long> tm(wn.n_todo * 16);
        CK(cudaMemcpy(tm.data(), wn.lz4_timing.p, tm.size() * 8, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < wn.n_todo; ++i) {
          const long long* q = &tm[i * 16];
          if (!q[3]) continue;  // not an LZ4 page (or the warp fallback)
          // [0] skim (phases 1-2), [1] phase 3, [2] phase 4 (warp path: k_page_matches' clocks)
          const double c[3] = {(double)(q[2] - q[0]), (double)(q[3] - q[2]),
                               q[12] ? (double)(q[12] - q[11]) : 0.0};
          for (int ph = 0; ph < 3; ++ph) lz4_phase_cycles[ph] = std::max(lz4_phase_cycles[ph], c[ph]);
        }
      }
      if (src_done) src_done(src_user, wn.epoch, wn.pos0, wn.n);  // its pages are on the device
      cur = nxt;
      served = 0;
      clouds += wn.n;
      for (size_t f = 0; f < outs.size(); ++f)
        for (uint64_t k = 0; k < wn.n; ++k) alg_bytes += wn.h_len[f * wn.n + k];
      alg_bytes += wn.in_payload_bytes;
      points_in += wn.in_points;
      payload_bytes += wn.in_payload_bytes;
      if (host_batches) {
        uint64_t first_bad = wn.n;
        for (uint64_t s = 0; s < wn.n; ++s)
          if (wn.h_status[s] != kOk) {
            first_bad = s;
            break;
          }
        const uint64_t B64 = g.batch_size;
        stage_host(wn, first_bad == wn.n ? wn.n : first_bad / B64 * B64);
      }
    }
    Wave& w = slots[cur];
    const uint32_t B = g.batch_size;
    const uint64_t s0 = (uint64_t)served * B;
    const uint64_t s1 = std::min<uint64_t>(s0 + B, w.n);
    const uint32_t nb = (uint32_t)(s1 - s0);
    for (uint64_t s = s0; s < s1; ++s)
      if (w.h_status[s] != kOk) {
        failed = true;
        fail_code = kWorkerPanic;
        fail_msg = op_message(w.h_status[s], w.h_op[s], w.h_where[s]);
        fail(fail_code, fail_msg);
      }
    std::memset(out, 0, sizeof(*out));
    out->epoch = w.epoch;
    out->batch_index = w.first_batch + served;
    out->n_samples = nb;
    out->n_fields = (uint32_t)outs.size();
    w.offsets.assign(outs.size(), std::vector<uint64_t>(nb + 1, 0));

    for (size_t f = 0; f < outs.size(); ++f) {
      pcp_field& pf = out->fields[f];
      std::snprintf(pf.name, sizeof(pf.name), "%s", outs[f].name.c_str());
      pf.kind = outs[f].kind;
      auto& off = w.offsets[f];
      const uint64_t b0 = field_offset(w, f, s0);
      bool uniform = true;
      for (uint32_t k = 0; k < nb; ++k) {
        off[k + 1] = field_offset(w, f, s0 + k + 1) - b0;
        if (w.h_len[f * w.n + s0 + k] != w.h_len[f * w.n + s0]) uniform = false;
      }
      pf.uniform = uniform ? 1 : 0;
      pf.nbytes = off[nb];
      pf.h_offsets = off.data();
      pf.d_ptr = const_cast<uint8_t*>(field_base(w, f)) + b0;
      if (host_batches) pf.h_ptr = w.h_out.as<uint8_t>() + w.h_base[f] + b0;
    }
    ++served;
    ++batches;
    items_emitted += nb;
    return kOk;
  }

  // ---- live reconfiguration (update_op_config) -----------------------------
  // {"slots": s, "wave_batches": k}: applied at the next wave boundary once
  // the waves in flight are served (content, order and seeds are independent
  // of both knobs).  Not while streaming from files (the reader's plan).
  void update_config(const std::string& text) {
    json o = json::parse(text, nullptr, false);
    if (o.is_discarded() || !o.is_object()) fail(kOutOfBounds, "config is not a JSON object");
    for (auto it = o.begin(); it != o.end(); ++it)
      if (it.key() != "slots" && it.key() != "wave_batches") fail(kUnknownOp, "knob '" + it.key() + "'");
    if (o.contains("slots")) {
      const int64_t v = o["slots"].get<int64_t>();
      if (v < 2 || v > 8) fail(kOutOfBounds, "slots outside [2, 8]");
    }
    if (o.contains("wave_batches") && o["wave_batches"].get<int64_t>() < 1)
      fail(kOutOfBounds, "wave_batches must be >= 1");
    if (stream_files) fail(kOutOfBounds, "not reconfigurable while streaming pages from files");
    for (auto it = o.begin(); it != o.end(); ++it) pending_cfg[it.key()] = it.value();
    has_pending = true;
  }

  void apply_config() {
    if (pending_cfg.contains("wave_batches")) {
      wave_batches = pending_cfg["wave_batches"].get<uint32_t>();
      plan_waves();
    }
    if (pending_cfg.contains("slots")) {
      const size_t want = pending_cfg["slots"].get<size_t>();
      CK(cudaStreamSynchronize(serve_stream));
      while (slots.size() > want) {
        destroy_slot(slots.back());
        slots.pop_back();
      }
      const size_t have = slots.size();
      slots.resize(want);
      for (size_t k = have; k < want; ++k) create_slot(slots[k]);
      n_slots = (uint32_t)want;
    }
    pending_cfg = json::object();
    has_pending = false;
    ++reconfigs;
  }

  // Pipeline::metrics (pipeline.hpp:140-149, pipeline.cpp:734-766) for the
  // device stage: the map nodes run as one fused kernel stage per wave
  // (busy = its device time), the source node is page CRC + decode, the sink
  // is the served wave; an "empty poll" is a next_batch that had to wait for
  // the device (the data-side signal of detect_bottleneck).
  const char* metrics() {
    const double up = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    json ops = json::array();
    ops.push_back({{"op_id", g.source_id}, {"kind", "source"},
                   {"num_workers", stream_files ? reader_threads : 1u}, {"items", clouds},
                   {"busy_seconds", (crc_kernel_ms + decode_kernel_ms) * 1e-3},
                   {"out_queue_size", 0}, {"out_queue_capacity", 0}});
    std::vector<uint32_t> map_nodes;
    for (const auto& m : g.maps)
      if (map_nodes.empty() || map_nodes.back() != m.node_id) map_nodes.push_back(m.node_id);
    const uint64_t in_flight = [&] {
      uint64_t k = 0;
      for (const auto& w : slots) k += w.launched ? 1 : 0;
      return k;
    }();
    for (uint32_t id : map_nodes)
      ops.push_back({{"op_id", id}, {"kind", "map"}, {"num_workers", (uint64_t)slots.size()}, {"items", clouds},
                     {"busy_seconds", (cloud_kernel_ms + vx_kernel_ms) * 1e-3 / map_nodes.size()},
                     {"out_queue_size", in_flight}, {"out_queue_capacity", (uint64_t)slots.size()}});
    const uint64_t ready = (cur >= 0 && served < slots[cur].n_batches) ? slots[cur].n_batches - served : 0;
    ops.push_back({{"op_id", g.batch_id}, {"kind", "batch"}, {"num_workers", 1}, {"items", items_emitted},
                   {"busy_seconds", csr_kernel_ms * 1e-3}, {"out_queue_size", ready},
                   {"out_queue_capacity", (uint64_t)slots.size() * cur_wave_batches}});
    json m{{"uptime_seconds", up},
           {"ops", ops},
           {"sink_polls", sink_polls},
           {"sink_empty_polls", sink_empty_polls},
           {"sink_size", ready},
           {"sink_capacity", (uint64_t)slots.size() * cur_wave_batches},
           {"batches_emitted", batches},
           {"items_emitted", items_emitted},
           {"slots", (uint64_t)slots.size()},
           {"wave_batches", cur_wave_batches},
           {"reconfigs", reconfigs}};
    metrics_json = m.dump();
    return metrics_json.c_str();
  }

  const char* stats() {
    json j{{"clouds", clouds},
           {"points_in", points_in},
           {"payload_bytes", payload_bytes},
           {"batches", batches},
           {"waves", waves_done},
           {"cloud_kernel_ms", cloud_kernel_ms},
           {"cloud_kernel_alg_bytes", alg_bytes},
           {"decode_kernel_ms", decode_kernel_ms},
           {"decode_kernel_alg_bytes", decode_alg_bytes},
           {"crc_kernel_ms", crc_kernel_ms},
           {"crc_kernel_alg_bytes", crc_alg_bytes},
           {"csr_kernel_ms", csr_kernel_ms},
           {"vx", vx_on},
           {"lz4_pj_waves", lz4_pj_waves},
           {"kernels", json{{"k_vx_*(voxel stage)", json{{"ms", vx_kernel_ms}, {"alg_bytes", vx_alg_bytes}}}}},
           {"csr_kernel_alg_bytes", csr_alg_bytes},
           {"serial", serial},
           {"block_pages_lz4", block_pages_lz4},
           {"block_pages_stored_raw", block_head.size() - block_pages_lz4},
           {"h2d_bytes", h2d_bytes},
           {"loaded_bytes", loaded_bytes},
           {"store_bytes", store_bytes},
           {"stream", stream_files},
           {"read_bytes", read_bytes},
           {"read_wait_ms", read_wait_ms},
           {"d2h_bytes", d2h_bytes},
           {"host_launch_ms", host_launch_ms},
           {"host_wait_ms", host_wait_ms},
           {"timeline", timeline},
           {"launches", launches},
           {"grid", grid},
           {"threads", threads},
           {"slots", (uint64_t)slots.size()},
           {"smem_bytes", smem},
           {"cloud_grid", grid},
           {"slots", (uint64_t)slots.size()},
           {"slab_bytes_per_slot", proto.gscratch_per_cta * (uint64_t)std::max(grid, grid_pre)},
           {"cloud_min_blocks", proto.min_blocks},
           {"fps_cluster", proto.fps_cluster},
           {"smem_mode", proto.smem_mode},
           {"cap_points", proto.cap_points},
           {"resident", resident},
           {"lz4_max_phase_cycles", lz4_phase_cycles}};
    if (op_timing && d_op_cycles.p) {  // summed over CTAs: [stage+decode, ops..., writes]
      std::vector<unsigned long long> oc(kMaxOps + 2);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(oc.data(), d_op_cycles.p, oc.size() * 8, cudaMemcpyDeviceToHost));
      j["voxel_phase_cycles"] = std::vector<unsigned long long>(oc.begin() + 10, oc.begin() + 15);
      oc.resize(proto.n_ops + 2);
      j["op_cycles"] = oc;
    }
    stats_json = j.dump();
    return stats_json.c_str();
  }
};


}  // namespace pcp

// =========================================================================
// C ABI
// =========================================================================
using namespace pcp;

extern "C" {

struct pcp_pipeline {
  pcp::Pipeline impl;
};

const char* pcp_last_error(void) { return g_err.c_str(); }

const char* pcp_errc_name(int status) { return errc_name(status); }

int pcp_device_info(int device, int* sm_count, int* cc_major, int* cc_minor) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) fail(kIoFailure, "no CUDA device");
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, device));
    *sm_count = p.multiProcessorCount;
    *cc_major = p.major;
    *cc_minor = p.minor;
  });
}

uint64_t pcp_mix_seed(uint64_t base, uint64_t epoch, uint64_t index, uint64_t op) {
  auto mix = [](uint64_t h, uint64_t v) {
    h += 0x9e3779b97f4a7c15ull + v;
    h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
    h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
    return h ^ (h >> 31);
  };
  uint64_t h = mix(base, 0x706370ull);
  h = mix(h, epoch);
  h = mix(h, index);
  return mix(h, op);
}

int pcp_map_kind_from_name(const char* name, int* kind) {
  return guarded([&] { *kind = map_kind_from_name(name ? name : ""); });
}

int pcp_crc32_ranges(const uint8_t* d_bytes, const uint64_t* d_off, const uint64_t* d_len,
                     uint32_t n, uint32_t* d_crc, void* stream) {
  return guarded([&] {
    auto st = (cudaStream_t)stream;
    DeviceCtx& c = device_ctx(st);
    CK(launch_crc_ranges(d_bytes, d_off, d_len, n, c.shift.as<uint32_t>(), d_crc, st));
  });
}

int pcp_decode_pages(const uint8_t* d_bytes, const uint64_t* d_page_off, uint32_t n_pages,
                     uint8_t* d_out, const uint64_t* d_out_off, const uint32_t* d_col_first,
                     const uint64_t* d_col_off, const uint64_t* d_col_len, int32_t* d_status,
                     void* stream) {
  return guarded([&] {
    auto st = (cudaStream_t)stream;
    DeviceCtx& c = device_ctx(st);
    if (!n_pages) return;
    // page heads → per-page LZ4 scratch slabs (convenience path: one D2H)
    std::vector<uint64_t> off(n_pages), sc_off(n_pages);
    CK(cudaMemcpyAsync(off.data(), d_page_off, n_pages * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    uint64_t total = 0;
    for (uint32_t i = 0; i < n_pages; ++i) {
      uint8_t head[kPageHeaderBytes];
      CK(cudaMemcpy(head, d_bytes + off[i], kPageHeaderBytes, cudaMemcpyDeviceToHost));
      uint64_t pay;
      std::memcpy(&pay, head + 9, 8);
      sc_off[i] = total;
      if (head[0] & kFlagOuterLz4) total = align16(total + lz4_scratch_bytes(std::min<uint64_t>(pay, 1ull << 32)));
    }
    c.scratch.ensure(total + 128 + n_pages * 8);
    uint64_t* d_sc_off = reinterpret_cast<uint64_t*>(c.scratch.as<uint8_t>() + align16(total + 64));
    CK(cudaMemcpyAsync(d_sc_off, sc_off.data(), n_pages * 8, cudaMemcpyHostToDevice, st));
    CK(launch_decode_pages(d_bytes, d_page_off, n_pages, d_out, d_out_off, d_col_first, d_col_off,
                           d_col_len, c.shift.as<uint32_t>(), d_sc_off, c.scratch.as<uint8_t>(),
                           d_status, st));
    CK(cudaStreamSynchronize(st));
  });
}

int pcp_apply_map(int kind, const char* params_json, const pcp_cloud_set* in,
                  const pcp_cloud_out* out, const uint64_t* d_seeds, int32_t* d_status,
                  void* stream) {
  return guarded([&] {
    auto st = (cudaStream_t)stream;
    DeviceCtx& ctx = device_ctx(st);
    if (!in || !out || !in->d_data) fail(kMissingField, "cloud set needs data");
    const uint32_t n = in->n_clouds;
    if (!n) return;
    std::vector<uint64_t> off(n + 1);
    CK(cudaMemcpyAsync(off.data(), in->d_offset, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    uint64_t max_n = 0;
    for (uint32_t i = 0; i < n; ++i) max_n = std::max<uint64_t>(max_n, off[i + 1] - off[i]);
    WaveArgs a;
    std::memset(&a, 0, sizeof(a));
    a.neg_zero = -0.0f;
    a.set_mode = 1;
    a.n_bytes_fields = kMaxBytesFields;
    a.role_data = 0;
    a.role_normal = in->d_normal ? 1 : -1;
    a.role_color = in->d_color ? 2 : -1;
    a.role_intensity = in->d_intensity ? 3 : -1;
    const uint8_t* srcs[8] = {(const uint8_t*)in->d_data, (const uint8_t*)in->d_normal,
                              (const uint8_t*)in->d_color, (const uint8_t*)in->d_intensity,
                              in->d_extra[0], in->d_extra[1], in->d_extra[2], in->d_extra[3]};
    uint8_t* dsts[8] = {(uint8_t*)out->d_data, (uint8_t*)out->d_normal, (uint8_t*)out->d_color,
                        (uint8_t*)out->d_intensity, out->d_extra[0], out->d_extra[1],
                        out->d_extra[2], out->d_extra[3]};
    const uint32_t elems[8] = {12, 12, 12, 4, in->extra_elem[0], in->extra_elem[1],
                               in->extra_elem[2], in->extra_elem[3]};
    for (int f = 0; f < 8; ++f) {
      if (!srcs[f]) continue;
      if (elems[f] == 0) fail(kOutOfBounds, "extra field with zero element size");
      a.tracked_mask |= 1u << f;
      a.set_src[f] = srcs[f];
      a.set_out[f] = dsts[f];
      a.set_elem[f] = elems[f];
      a.field_cap[f] = elems[f];
    }
    OpDesc& op = a.ops[0];
    op.kind = kind;
    json params = (params_json && *params_json) ? json::parse(params_json, nullptr, false) : json::object();
    if (params.is_discarded()) fail(kOutOfBounds, "params are not valid JSON");
    parse_op_params(op, params, [&](const std::string& nm) -> int {
      static const char* names[8] = {"data", "normal", "color", "intensity",
                                     "extra0", "extra1", "extra2", "extra3"};
      for (int f = 0; f < 8; ++f)
        if (nm == names[f] && srcs[f]) return f;
      return -1;
    });
    if (kind != kNormalize && kind != kTranslate && kind != kJitter && kind != kRotate &&
        kind != kRandomScale && kind != kFlipYz && kind != kColorAugment && kind != kRandomCrop &&
        kind != kDownsample && kind != kFps && kind != kRangeCrop && kind != kVoxel)
      fail(kUnknownOp, "unknown map kind " + std::to_string(kind));
    a.n_ops = 1;
    a.cap_points = (uint32_t)std::max<uint64_t>({max_n, (uint64_t)std::max<int64_t>(op.num_points, 0), 1});
    a.set_out_cap = out->cap_points;
    a.n_samples = n;
    a.set_offset = in->d_offset;
    a.set_seeds = d_seeds;
    a.set_count = out->d_count;
    a.sample_status = d_status;
    a.voxel_scratch = kind == kVoxel ? 1 : 0;
    a.set_voxel_count = out->d_voxel_count;
    a.count_out = -1;
    cudaDeviceProp prop;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaGetDeviceProperties(&prop, dev));
    const size_t fixed = cloud_smem_fixed();
    plan_fps_cluster(a, 512);
    const size_t smem = fixed + plan_buffers(a, false, prop.sharedMemPerBlockOptin - fixed);
    CK(set_apply_smem(smem));
    int grid = ctx.sms * 2;
    if (a.fps_cluster > 1) {
      int clusters = 0;
      CK(occupancy_cloud_clusters(&clusters, 512, smem, a.fps_cluster, true));
      if (clusters < 1) fail(kOutOfBounds, "no room for a cluster of " + std::to_string(a.fps_cluster) + " CTAs");
      grid = std::min<int>(clusters, (int)n) * (int)a.fps_cluster;
    }
    if (a.gscratch_per_cta) {
      if (a.fps_cluster <= 1) grid = std::min<int>(grid, (int)n);
      ctx.scratch.ensure(a.gscratch_per_cta * grid);
      a.gscratch = ctx.scratch.as<uint8_t>();
    }
    CK(launch_apply_set(a, grid, 512, smem, st));
  });
}

namespace {
int write_dataset_impl(const char* out_dir, const char* stem, const char* schema_json, const uint8_t* tlv,
                       size_t tlv_len, uint32_t n_samples, uint32_t slice_count, uint32_t group_size,
                       uint32_t n_threads, int device);
}

int pcp_write_dataset(const char* out_dir, const char* stem, const char* schema_json,
                      const uint8_t* tlv, size_t tlv_len, uint32_t n_samples,
                      uint32_t slice_count, uint32_t group_size, uint32_t n_threads) {
  return write_dataset_impl(out_dir, stem, schema_json, tlv, tlv_len, n_samples, slice_count, group_size,
                            n_threads, -1);
}

int pcp_write_dataset_device(const char* out_dir, const char* stem, const char* schema_json,
                             const uint8_t* tlv, size_t tlv_len, uint32_t n_samples,
                             uint32_t slice_count, uint32_t group_size, int device) {
  return write_dataset_impl(out_dir, stem, schema_json, tlv, tlv_len, n_samples, slice_count, group_size,
                            16, device);
}

namespace {
int write_dataset_impl(const char* out_dir, const char* stem, const char* schema_json, const uint8_t* tlv,
                       size_t tlv_len, uint32_t n_samples, uint32_t slice_count, uint32_t group_size,
                       uint32_t n_threads, int device) {
  return guarded([&] {
    const auto schema = schema_from_json(schema_json);
    std::vector<SampleIn> samples(n_samples);
    size_t pos = 0;
    auto need = [&](size_t k) {
      if (pos + k > tlv_len) fail(kSchemaMismatch, "sample stream truncated");
    };
    for (uint32_t i = 0; i < n_samples; ++i) {
      need(4);
      uint32_t nf;
      std::memcpy(&nf, tlv + pos, 4);
      pos += 4;
      samples[i].values.assign(schema.size(), {});
      std::vector<bool> seen(schema.size(), false);
      for (uint32_t f = 0; f < nf; ++f) {
        need(2);
        uint16_t nl;
        std::memcpy(&nl, tlv + pos, 2);
        pos += 2;
        need(nl + 9);
        std::string name(reinterpret_cast<const char*>(tlv + pos), nl);
        pos += nl;
        const uint8_t kind = tlv[pos++];
        uint64_t nb;
        std::memcpy(&nb, tlv + pos, 8);
        pos += 8;
        need(nb);
        size_t fi = 0;
        while (fi < schema.size() && schema[fi].name != name) ++fi;
        if (fi == schema.size() || schema[fi].kind != (int32_t)kind)
          fail(kSchemaMismatch, "field '" + name + "' not in schema or mistyped");
        samples[i].values[fi].assign(tlv + pos, tlv + pos + nb);
        seen[fi] = true;
        pos += nb;
      }
      for (size_t f = 0; f < schema.size(); ++f)
        if (!seen[f]) fail(kSchemaMismatch, "missing field '" + schema[f].name + "'");
    }
    write_dataset(schema, samples, slice_count, group_size, out_dir, stem, n_threads ? n_threads : 8, device);
  });
}
}  // namespace

int pcp_pipeline_open(const char* primary, const char* graph_json, const uint64_t* ids,
                      uint64_t n_ids, int device, const char* options, pcp_pipeline** out) {
  *out = nullptr;
  return guarded([&] {
    auto p = std::make_unique<pcp_pipeline>();
    p->impl.open(primary, graph_json, ids, n_ids, device, options ? options : "");
    *out = p.release();
  });
}

int pcp_pipeline_open_source(const uint8_t* header, size_t header_len, const char* graph_json,
                             const uint64_t* ids, uint64_t n_ids, int device, const char* options,
                             pcp_page_source_fn read, pcp_wave_done_fn done, void* user,
                             pcp_pipeline** out) {
  *out = nullptr;
  return guarded([&] {
    if (!header || !read) fail(kOutOfBounds, "header bytes and a page source are required");
    auto p = std::make_unique<pcp_pipeline>();
    const std::vector<uint8_t> hb(header, header + header_len);
    p->impl.src_header = &hb;
    p->impl.src_read = read;
    p->impl.src_done = done;
    p->impl.src_user = user;
    p->impl.open("", graph_json, ids, n_ids, device, options ? options : "");
    p->impl.src_header = nullptr;
    *out = p.release();
  });
}

int pcp_pipeline_next_batch(pcp_pipeline* p, pcp_batch* out, int* eos) {
  return guarded([&] { p->impl.next_batch(out, eos); });
}

void* pcp_pipeline_stream(pcp_pipeline* p) { return p->impl.serve_stream; }

const char* pcp_pipeline_stats(pcp_pipeline* p) { return p->impl.stats(); }

const char* pcp_pipeline_metrics(pcp_pipeline* p) { return p->impl.metrics(); }

int pcp_pipeline_update_config(pcp_pipeline* p, const char* config_json) {
  return guarded([&] { p->impl.update_config(config_json ? config_json : ""); });
}

void pcp_pipeline_close(pcp_pipeline* p) { delete p; }

int pcp_malloc(void** d, size_t n) {
  return guarded([&] { CK(cudaMalloc(d, n)); });
}
int pcp_free(void* d) {
  return guarded([&] { CK(cudaFree(d)); });
}
int pcp_memcpy_h2d(void* d, const void* h, size_t n, void* st) {
  return guarded([&] {
    CK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, (cudaStream_t)st));
    CK(cudaStreamSynchronize((cudaStream_t)st));
  });
}
int pcp_memcpy_d2h(void* h, const void* d, size_t n, void* st) {
  return guarded([&] {
    CK(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, (cudaStream_t)st));
    CK(cudaStreamSynchronize((cudaStream_t)st));
  });
}
int pcp_memcpy_d2h_async(void* h, const void* d, size_t n, void* st) {
  return guarded([&] { CK(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, (cudaStream_t)st)); });
}
int pcp_stream_sync(void* st) {
  return guarded([&] { CK(cudaStreamSynchronize((cudaStream_t)st)); });
}

}  // extern "C"
