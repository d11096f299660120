#!/usr/bin/env python
"""bench.py — PcRecord → training-batch throughput on B200 (BASELINE.json metric:
point clouds/s and Mpoints/s per GPU and for N GPUs, next to the reference CPU
pipeline, with the HBM-roofline fraction of the dominant kernel).

  python bench.py [--gpus N --steps K --warmup W] [--config s3dis] [--quantized]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)
  python bench.py --impl reference ...                (the reference CPU arm)

Default workload (N=1 headline): C3 S3DIS-shaped rooms — BASELINE.json's
metric names no config, so the line is quoted on the largest single-GPU
configuration; the other four configs are under --config.

A step = one pass of the hot path (page CRC + decode, record parse, the
config's op chain, batch assembly) over this rank's shard of the synthetic
dataset (record-sharded by slice, no collective on the data path).
`value`: pages resident in HBM before the timed region.  `e2e`: pages in
pinned host memory, per-wave H2D of the pages and every batch delivered in
pinned host memory (host_batches: one D2H per field per wave) inside the
timed region, through the C ABI (pcp_pipeline_*).  Inputs per step exceed
the 126 MB L2, so no flush is needed between steps.
`roofline`: per-kernel times from a separate serial pass (option "serial":
one wave in flight, CUDA events around each kernel on the wave's stream), so
every kernel's time is its own and the kernel times sum to at most the
serial step time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# workload per config: generator, points, clouds per GPU, group size, batch
CONFIGS = {
    "shapenet_part": dict(gen="shapenet", kw={"n_points": 2048}, clouds=16384, group=64, batch=32, cpu_sample=4096,
                          points=2048, desc="ShapeNet-part-shaped 2048-pt clouds + per-point seg "
                          "labels: normalize, downsample 1024 (+seg), random_scale, shuffle; B 32"),
    "modelnet40": dict(gen="modelnet", kw={"n_points": 10000}, clouds=2048, group=32, group_q=8, batch=32,
                       cpu_sample=256,
                       points=10000, desc="ModelNet40-shaped 10k-pt clouds + normals: normalize, "
                       "FPS 1024, rotate, jitter; B 32"),
    "kitti": dict(gen="kitti", kw={}, clouds=512, group=16, group_q=1, batch=4, points=120000, cpu_sample=128,
                  desc="KITTI-shaped ~120k-pt XYZI frames: range crop, voxel 0.05 m (+counts), "
                  "rotate, flip_yz; B 4 (CSR batches)"),
    "s3dis": dict(gen="s3dis", kw={"mean_points": 1_000_000}, clouds=256, group=1, batch=4, cpu_sample=128,
                  points=1_000_000, desc="S3DIS-shaped ~1M-pt XYZRGB rooms: grid 0.04 m, "
                  "random_crop, downsample 4096; B 4"),
    "scannet": dict(gen="scannet", kw={}, clouds=192, group=4, group_q=1, batch=4, points=275000, cpu_sample=64,
                    desc="ScanNet-shaped 50k-500k-pt XYZRGB scenes: grid 0.02 m, downsample "
                    "40000, FPS 20000; B 4"),
}
CHAIN_OF = {k: k for k in CONFIGS}
REF_OPS = {"normalize", "translate", "jitter", "rotate", "random_scale", "flip_yz",
           "color_augment", "random_crop", "downsample"}
SLICES = 8
DEFAULT_CONFIG = "s3dis"


def load_synth():
    """paper_2603_16945_b200/synth.py (pure numpy) loaded by path, so the
    reference arm never imports the package (nor maps its CUDA library)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "pcp_synth", os.path.join(ROOT, "paper_2603_16945_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def gen_samples(cfg, n, quantized, first=0, chunk=2048):
    synth = load_synth()
    gen = getattr(synth, cfg["gen"])
    schema, samples = None, []
    for f in range(first, first + n, chunk):
        schema, s = gen(min(chunk, first + n - f), quantized=quantized, first=f, **cfg["kw"])
        samples += s
    return schema, samples


def env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def dataset(cfg_name, cfg, world, quantized, rank, barrier):
    """The synthetic dataset on local disk, written with the library's writer
    (byte-identical to the reference's write_dataset, tests/test_host.py).
    N = 1: clouds_per_gpu clouds in 8 slices.  N > 1: rank r's shard of the
    global set -- clouds [r*C, (r+1)*C), generated with their global seeds --
    written by rank r as its own dataset, all ranks in parallel (one process
    would hold and write N x 6 GB of S3DIS rooms serially), so each rank
    reads only its own shard and no data crosses ranks."""
    from paper_2603_16945_b200 import write_dataset
    C = cfg["clouds"]
    d = f"/tmp/pcp_bench_{cfg_name}_{'q' if quantized else 'raw'}_{C}x{world}_g{cfg['group']}"
    if world > 1:
        d += f"_r{rank}"
    primary = os.path.join(d, "ds.pcrecord")
    schema, samples = gen_samples(cfg, C, quantized, first=rank * C)
    write_dataset(d, "ds", schema, samples, slice_count=SLICES, group_size=cfg["group"],
                  n_threads=max(1, min(32, (os.cpu_count() or 1) // world)))
    del samples
    barrier()
    return primary


def reference_dataset(cfg_name, cfg, quantized, n):
    """The reference arm's input: n clouds of the same workload written by the
    REFERENCE writer (oracle/_ref write_dataset, format.cpp:499-610)."""
    from oracle.ffi import Ref
    d = f"/tmp/pcp_refarm_{cfg_name}_{'q' if quantized else 'raw'}_{n}_g{cfg['group']}"
    schema, samples = gen_samples(cfg, n, quantized)
    return Ref().write_dataset(d, "ds", schema, samples, slice_count=SLICES, group_size=cfg["group"])


class Clocks:
    """SM clocks and throttle reasons sampled every 20 ms during the timed
    region (NVML; falls back to nvidia-smi -lms 200)."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, dev):
        self.dev, self.rows, self.stop, self.t, self.p = dev, [], False, None, None

    def _nvml(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self.stop:
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((sm, mx, rs))
            time.sleep(0.02)

    def __enter__(self):
        try:
            import pynvml  # noqa: F401
            self.t = threading.Thread(target=self._nvml, daemon=True)
            self.t.start()
        except Exception:
            try:
                q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active")
                self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                           "--format=csv,noheader,nounits", "-lms", "200"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._smi, daemon=True)
                self.t.start()
            except OSError:
                pass
        return self

    def _smi(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            try:
                self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
            except (ValueError, IndexError):
                pass

    def __exit__(self, *a):
        self.stop = True
        if self.p:
            self.p.terminate()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic(workload, kernel):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        k = s.get(workload, {}).get(kernel, {})
        return k.get("dram_bytes_per_launch"), k.get("clouds_per_launch")
    except (OSError, ValueError):
        return None, None


def graph_for(cfg_name, cfg, workers=1):
    synth = load_synth()
    return synth.graph(synth.CHAINS[CHAIN_OF[cfg_name]], batch_size=cfg["batch"], base_seed=42,
                       workers=workers)


APPC_OPS = {"fps", "voxel", "grid_subsample", "range_crop"}


# cpu_sample: clouds per reference step.  run_benchmark excludes the first
# batch from its clock, so a step needs several clouds per host thread (a
# sample of one cloud per worker finishes all clouds together and leaves the
# clock almost nothing: 16 ScanNet scenes on 16 threads read 488 K clouds/s).


def cpu_reference(primary, graph, sample_ids, steps, warmup):
    """The reference CPU pipeline on a bounded sample of the same workload,
    with all host threads, run_benchmark timing (bench.cpp:43-96: items over
    the cost time, warm-up batch excluded from the clock).

    Chains of reference ops run in the reference Pipeline (oracle/_ref: the
    unmodified reference sources) -> kind "reference".  Chains with App. C
    ops (fps / voxel / grid / range crop: absent from the reference) run the
    same reference Pipeline, whose SourceFn applies the chain up to the last
    App. C op after read_sample (App. C ops in the C restatement, reference
    ops in the reference apply_map) on every host thread, the remaining
    reference ops in its map workers -> kind "port".  Returns
    (clouds/s median, cores, kind, description)."""
    from oracle.ffi import Ref
    ref = Ref()
    ncpu = os.cpu_count() or 1
    g = json.loads(json.dumps(graph))
    maps = [o for o in g["ops"] if o["kind"] == "map"]
    last_c = max([i for i, o in enumerate(maps) if o["map"] in APPC_OPS], default=-1)
    src = g["ops"][0]
    for o in maps:
        o["num_workers"] = ncpu
    if last_c < 0:
        src["num_workers"] = min(4, ncpu)
        run = lambda: ref.bench_pipeline(primary, g, repeats=1, ids=sample_ids)
        kind, how = "reference", f"reference Pipeline (oracle/_ref), {min(4, ncpu)} source + {ncpu} map workers"
    else:
        src["num_workers"] = ncpu
        prefix = [{"map": o["map"], "params": o.get("params", {}), "op_id": o["id"]} for o in maps[:last_c + 1]]
        g2 = dict(g, ops=[src] + maps[last_c + 1:] + [o for o in g["ops"] if o["kind"] in ("batch", "sink")])
        run = lambda: ref.bench_composed(primary, g2, prefix, repeats=1, ids=sample_ids)
        kind = "port"
        how = (f"reference Pipeline (oracle/_ref) with {ncpu} source workers whose SourceFn runs "
               f"read_sample + {'/'.join(p['map'] for p in prefix)} (App. C ops in the C restatement, "
               f"reference ops in reference apply_map)"
               + (f", then {ncpu} map workers for {'/'.join(o['map'] for o in maps[last_c + 1:])}"
                  if maps[last_c + 1:] else ""))
    vals = []
    for i in range(warmup + steps):
        r = run()
        if i >= warmup:
            vals.append(r["items"] / r["cost_time_s"])
    return statistics.median(vals), ncpu, kind, how


def kernel_pass(P, primary, g, ids, local, steps):
    """Per-kernel device time without overlap: a fresh pipeline with option
    "serial" (one wave in flight), CUDA events around every kernel on the
    wave's stream.  Returns ({kernel: {ms_per_step, alg_bytes_per_step}},
    serial ms per step)."""
    import torch
    p = P.Pipeline(primary, g, ids=ids, device=local, epochs=steps, resident=True, serial=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while p.next_batch_raw() is not None:
        pass
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    st = p.stats()
    p.close()
    out = {}
    names = {"k_crc_windows": "crc", "k_page_decode+k_page_matches": "decode", "k_cloud": "cloud",
             "k_wave_offsets+k_compact_wave": "csr"}
    for k, key in names.items():
        ms = st[f"{key}_kernel_ms"]
        by = st[f"{key}_kernel_alg_bytes"]
        if ms > 0:
            out[k] = {"ms_per_step": ms / steps, "alg_bytes_per_step": by / steps}
    for k, v in st.get("kernels", {}).items():  # further timed kernels (name -> ms, alg bytes)
        if v["ms"] > 0:
            out[k] = {"ms_per_step": v["ms"] / steps, "alg_bytes_per_step": v["alg_bytes"] / steps}
    return out, e0.elapsed_time(e1) / steps, st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--quantized", action="store_true", help="LZ4 page variant")
    ap.add_argument("--clouds-per-gpu", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-pass", action="store_true")
    ap.add_argument("--e2e-no-d2h", action="store_true", help="diagnostics: e2e without the batch reads")
    ap.add_argument("--cpu-sample", type=int, default=0, help="clouds per CPU step")
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch size (diagnostics)")
    ap.add_argument("--group", type=int, default=0, help="override the writer's group size (samples per page)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    # quantized pages are one LZ4 block each, decoded by one serial token chain:
    # those variants are written with ~2 MB pages where the config allows
    # (SURVEY.md §7 hard part 1: "choose G per config for the quantized variant")
    if args.quantized and "group_q" in cfg:
        cfg["group"] = cfg["group_q"]
    if args.group:
        cfg["group"] = args.group
    if args.batch:
        cfg["batch"] = args.batch
    if args.clouds_per_gpu:
        cfg["clouds"] = args.clouds_per_gpu
    rank, world, local = env()
    coords = "1 mm-quantised coordinates" if args.quantized else "raw float32 coordinates"
    config = {"workload": args.config, "desc": cfg["desc"], "variant": coords,
              "clouds_per_gpu_per_step": cfg["clouds"], "points_per_cloud": cfg["points"],
              "batch": cfg["batch"], "group_size": cfg["group"], "slices": SLICES,
              "parallelism": (f"record-sharded: rank r owns clouds [r*C, (r+1)*C) of the global set as "
                              f"its own dataset, {world} independent pipelines" if world > 1 else
                              "1 pipeline over all 8 slices"),
              "l2": "inputs per step > 126 MB L2 (no flush needed)"}
    metric = "point clouds/sec (PcRecord -> training batch)"
    cpu_sample = args.cpu_sample or cfg["cpu_sample"]

    if args.impl == "reference":
        if rank != 0:
            return
        # input written by the reference's own writer; the reference arm maps
        # no library of this repo
        primary = reference_dataset(args.config, cfg, args.quantized, cpu_sample)
        g = graph_for(args.config, cfg)
        v, ncpu, kind, how = cpu_reference(primary, g, None, args.steps, args.warmup)
        config["clouds_per_gpu_per_step"] = cpu_sample
        line = {"metric": metric, "value": v, "unit": "clouds/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded generators, paper_2603_16945_b200/synth.py; pages written by "
                        "the reference write_dataset)", "config": config,
                "mpoints_per_sec": v * cfg["points"] / 1e6,
                "cpu_baseline": {"value": v, "unit": "clouds/s", "cores": ncpu, "kind": kind,
                                 "sample": f"{cpu_sample} clouds of the workload per step; {how}"},
                "e2e": {"value": v, "unit": "clouds/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        if args.config == "shapenet_part":
            line["note"] = "reference downsample ignores the 'gather' extension (seg stays unmoved)"
        try:  # the reference arm must map no library of this repo
            with open("/proc/self/maps") as f:
                mapped = sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")})
            line["mapped_repo_libraries"] = [m for m in mapped if m.startswith(ROOT) and "/oracle/" not in m]
        except OSError:
            pass
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    if os.environ.get("PCP_BENCH_SHARED_GPU"):
        # plumbing test only (tests/test_gpu_bench_multirank.py): every rank on
        # cuda:0 with gloo collectives -- ranks share one GPU, so its numbers
        # are not a measurement
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if os.environ.get("PCP_BENCH_SHARED_GPU"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        barrier = dist.barrier
    else:
        barrier = lambda: None
    import paper_2603_16945_b200 as P
    from paper_2603_16945_b200 import shard
    primary = dataset(args.config, cfg, world, args.quantized, rank, barrier)
    idx = shard.read_index(primary)
    ids = None  # the rank's dataset is its shard
    g = graph_for(args.config, cfg)

    def timed(resident, steps, d2h):
        # d2h: host_batches -- every batch delivered in pinned host memory, as the
        # reference's Pipeline::next_batch returns host Batches (one D2H per field
        # per wave inside the library, the host waits for it before serving)
        p = P.Pipeline(primary, g, ids=ids, device=local, epochs=steps, resident=resident,
                       host_batches=d2h)
        st0 = p.stats()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(local) as ck:
            e0.record()
            nb = 0
            # the bare C-ABI loop (pcp_pipeline_next_batch), as a C++ GpuPipeline
            # would run it: no per-batch Python objects
            while True:
                b = p.next_batch_raw()
                if b is None:
                    break
                nb += 1
            torch.cuda.synchronize()
            e1.record()
            e1.synchronize()
        ms = e0.elapsed_time(e1)
        st1 = p.stats()
        p.close()
        return ms, st0, st1, nb, st1["d2h_bytes"] - st0["d2h_bytes"], ck.summary()

    # warm-up (W steps), then K timed steps on a fresh pipeline
    timed(True, args.warmup, False)
    ms, st0, st1, nb, _, clocks = timed(True, args.steps, False)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    clouds_rank = st1["clouds"] - st0["clouds"]
    points_rank = st1["points_in"] - st0["points_in"]
    tot = torch.tensor([clouds_rank, points_rank], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot)
    clouds_all, points_all = float(tot[0]), float(tot[1])
    value = clouds_all / (ms_max / 1e3)
    pages = {"block_pages_lz4": st1.get("block_pages_lz4"), "block_pages_stored_raw": st1.get("block_pages_stored_raw")}
    config["variant"] += (f"; block pages: {pages['block_pages_lz4']} LZ4, "
                          f"{pages['block_pages_stored_raw']} stored-raw")

    roof = None
    if not args.no_kernel_pass:
        # roofline of the dominant kernel: per-kernel device time from the
        # serial pass (no overlap between waves), algorithmic bytes per kernel
        # over that time, against the burst HBM peak
        peak, peak_kind = peaks()
        ksteps = max(1, min(args.steps, 3))
        kern, serial_ms, sst = kernel_pass(P, primary, g, ids, local, ksteps)
        for k, v in kern.items():
            v["achieved_gbs"] = v["alg_bytes_per_step"] / (v["ms_per_step"] / 1e3) / 1e9
            v["share_of_serial_step"] = v["ms_per_step"] / serial_ms
        dom = max(kern, key=lambda k: kern[k]["ms_per_step"])
        waves = max(1, sst["waves"]) / ksteps  # waves per step
        alg_per_launch = kern[dom]["alg_bytes_per_step"] / waves
        dram, cap_clouds = ncu_traffic(args.config + ("_q" if args.quantized else ""), dom)
        if dram is not None and cap_clouds:  # capture wave -> this run's wave (per-cloud traffic)
            dram = dram / cap_clouds * (clouds_rank / args.steps / waves)
        roof = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["achieved_gbs"], "peak": peak,
                "unit": "GB/s", "frac": kern[dom]["achieved_gbs"] / peak,
                "peak_kind": f"{peak_kind} burst copy bandwidth (kernel timed alone)",
                "traffic": dram, "alg_bytes_per_launch": alg_per_launch,
                "serial_ms_per_step": serial_ms, "kernels": kern,
                "timing": "serial pass (option serial: one wave in flight), CUDA events around each "
                          "kernel on the wave stream; kernel ms per step sum to <= serial_ms_per_step"}
        if dram is not None and alg_per_launch:
            roof["traffic_over_alg"] = dram / alg_per_launch
        if dom == "k_page_decode+k_page_matches":
            roof["note"] = ("latency-bound: one serial LZ4 token/match chain per page "
                            "(DESIGN.md 4.2); HBM fraction reported for completeness")
    e2e = None
    if not args.no_e2e:
        timed(False, 1, True)  # untimed: fills the library's pinned-buffer pool
        ems, est0, est1, enb, d2h, _ = timed(False, args.steps, not args.e2e_no_d2h)
        te = torch.tensor([ems], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        if os.environ.get("PCP_BENCH_DEBUG"):
            print("e2e stats:", {k: est1[k] - est0[k] for k in ("cloud_kernel_ms", "decode_kernel_ms", "waves",
                                                               "h2d_bytes", "host_launch_ms", "host_wait_ms")}, "ms", ems,
                  "| resident:", {k: st1[k] - st0[k] for k in ("cloud_kernel_ms", "decode_kernel_ms", "waves",
                                                              "host_launch_ms", "host_wait_ms")},
                  "ms", ms, file=sys.stderr)
            for row in est1.get("timeline", []):
                print("wave h2d %.2f-%.2f decode %.2f-%.2f cloud %.2f-%.2f done %.2f host %.2f" % tuple(row),
                      file=sys.stderr)
        e_clouds = est1["clouds"] - est0["clouds"]
        tc = torch.tensor([e_clouds], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tc)
        e2e = {"value": float(tc.item()) / (float(te.item()) / 1e3), "unit": "clouds/s",
               "h2d_bytes_per_step": (est1["h2d_bytes"] - est0["h2d_bytes"]) // args.steps,
               "d2h_bytes_per_step": d2h // args.steps,
               "path": "pcp_pipeline_open(resident=false, host_batches=true) + "
                       "pcp_pipeline_next_batch: pages H2D from pinned host memory each wave, "
                       "every batch field delivered in pinned host memory (pcp_field.h_ptr)"}
        # the e2e bound: page bytes over PCIe against a plain pinned H2D copy
        # measured now on this box (256 MiB x 4)
        h2d_total = est1["h2d_bytes"] - est0["h2d_bytes"]
        hb = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
        db = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        db.copy_(hb, non_blocking=True)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(4):
            db.copy_(hb, non_blocking=True)
        c1.record()
        c1.synchronize()
        peak_h2d = 4 * (256 << 20) / (c0.elapsed_time(c1) / 1e3) / 1e9
        del hb, db
        e2e["pcie"] = {"h2d_gbs": h2d_total / (ems / 1e3) / 1e9, "h2d_peak_gbs": peak_h2d,
                       "frac": h2d_total / (ems / 1e3) / 1e9 / peak_h2d,
                       "d2h_gbs": d2h / (ems / 1e3) / 1e9}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ids_cpu = np.arange(min(cpu_sample, len(idx)), dtype=np.uint64)
        v, ncpu, kind, how = cpu_reference(primary, g, ids_cpu, 1, 0)
        cpu = {"value": v, "unit": "clouds/s", "cores": ncpu, "kind": kind,
               "sample": f"{len(ids_cpu)} clouds of the same dataset; {how}"}
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "clouds/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded generators, paper_2603_16945_b200/synth.py)",
                "config": config, "mpoints_per_sec": points_all / (ms_max / 1e3) / 1e6,
                "per_gpu_clouds_per_sec": value / world, "roofline": roof,
                "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
                "gpu_launches": st1["launches"] - st0["launches"],
                "k_cloud_launch": {k: st1.get(k) for k in ("cloud_grid", "cloud_min_blocks", "smem_bytes",
                                                             "smem_mode", "fps_cluster", "slots",
                                                             "slab_bytes_per_slot")},
                "batches_per_step": nb / args.steps}
        if "op_cycles" in st1:  # PCP_OP_TIMING=1 diagnostics: share of k_cloud CTA time
            oc = st1["op_cycles"]
            synth = load_synth()
            names = (["stage+decode"] + [o if isinstance(o, str) else o[0]
                                         for o in synth.CHAINS[CHAIN_OF[args.config]]] + ["writes"])
            tot_c = max(1, sum(oc))
            line["op_cycle_share"] = {n: round(c / tot_c, 4) for n, c in zip(names, oc)}
            if "voxel_phase_cycles" in st1:
                vp = st1["voxel_phase_cycles"]
                line["voxel_phase_share"] = dict(zip(["origin+extent", "keys", "sort", "segments", "means"],
                                                     [round(v / tot_c, 4) for v in vp]))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
