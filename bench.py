#!/usr/bin/env python
"""bench.py — PcRecord → training-batch throughput on B200 (BASELINE.json metric:
point clouds/s and Mpoints/s per GPU and for N GPUs, next to the reference CPU
pipeline, with the HBM-roofline fraction of the dominant kernel).

  python bench.py [--gpus N --steps K --warmup W] [--config shapenet_part]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)
  python bench.py --impl reference ...                (the reference CPU arm)

A step = one pass of the hot path (page CRC + decode, record parse, the
config's op chain, batch assembly) over this rank's shard of the synthetic
dataset (record-sharded by slice, no collective on the data path).
`value`: pages resident in HBM before the timed region.  `e2e`: pages in
pinned host memory, per-wave H2D of the pages and every batch delivered in
pinned host memory (host_batches: one D2H per field per wave) inside the
timed region, through the C ABI (pcp_pipeline_* ).  Inputs per step exceed
the 126 MB L2, so no flush is needed between steps.
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
    "shapenet_part": dict(gen="shapenet", kw={"n_points": 2048}, clouds=16384, group=64, batch=32,
                          points=2048, desc="ShapeNet-part-shaped 2048-pt clouds + per-point seg "
                          "labels: normalize, downsample 1024 (+seg), random_scale, shuffle; B 32"),
    "modelnet40": dict(gen="modelnet", kw={"n_points": 10000}, clouds=2048, group=32, batch=32,
                       points=10000, desc="ModelNet40-shaped 10k-pt clouds + normals: normalize, "
                       "FPS 1024, rotate, jitter; B 32"),
    "kitti": dict(gen="kitti", kw={}, clouds=512, group=16, batch=4, points=120000,
                  desc="KITTI-shaped ~120k-pt XYZI frames: range crop, voxel 0.05 m (+counts), "
                  "rotate, flip_yz; B 4 (CSR batches)"),
    "s3dis": dict(gen="s3dis", kw={"mean_points": 1_000_000}, clouds=256, group=1, batch=4,
                  points=1_000_000, desc="S3DIS-shaped ~1M-pt XYZRGB rooms: grid 0.04 m, "
                  "random_crop, downsample 4096; B 4"),
    "scannet": dict(gen="scannet", kw={}, clouds=192, group=4, batch=4, points=275000,
                    desc="ScanNet-shaped 50k-500k-pt XYZRGB scenes: grid 0.02 m, downsample "
                    "40000, FPS 20000; B 4"),
}
CHAIN_OF = {k: k for k in CONFIGS}
REF_OPS = {"normalize", "translate", "jitter", "rotate", "random_scale", "flip_yz",
           "color_augment", "random_crop", "downsample"}
SLICES = 8


def env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def dataset(cfg_name, cfg, world, quantized, rank, barrier):
    """Rank 0 writes the synthetic dataset (clouds_per_gpu x world clouds,
    8 slices) to local disk; every rank then opens it."""
    from paper_2603_16945_b200 import synth, write_dataset
    d = f"/tmp/pcp_bench_{cfg_name}_{'q' if quantized else 'raw'}_{cfg['clouds']}x{world}"
    primary = os.path.join(d, "ds.pcrecord")
    if rank == 0:
        n = cfg["clouds"] * world
        gen = getattr(synth, cfg["gen"])
        chunk = 2048
        schema, samples = None, []
        for first in range(0, n, chunk):
            schema, s = gen(min(chunk, n - first), quantized=quantized, first=first, **cfg["kw"])
            samples += s
        write_dataset(d, "ds", schema, samples, slice_count=SLICES, group_size=cfg["group"],
                      n_threads=min(32, os.cpu_count() or 1))
        del samples
    barrier()
    return primary


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
    from paper_2603_16945_b200 import synth
    return synth.graph(synth.CHAINS[CHAIN_OF[cfg_name]], batch_size=cfg["batch"], base_seed=42,
                       workers=workers)


def cpu_reference(primary, graph, sample_ids, steps, warmup):
    """CPU baseline on a bounded sample of the same dataset.

    Graphs made only of reference ops run in the reference Pipeline
    (oracle/_ref: unmodified reference sources) with all host threads,
    run_benchmark-style timing (bench.cpp:43-96) -> kind "reference".
    Graphs with App. C ops (fps / voxel / grid / range crop — absent from the
    reference) run reference read_sample + reference ops + the C restatement
    for the rest, one thread -> kind "port"."""
    from oracle.ffi import Orc, Ref
    ref = Ref()
    ncpu = os.cpu_count() or 1
    g = json.loads(json.dumps(graph))
    steps_ops = [(o["map"], o.get("params", {}), o["id"]) for o in g["ops"] if o["kind"] == "map"]
    if all(k in REF_OPS for k, _, _ in steps_ops):
        for o in g["ops"]:
            if o["kind"] == "source":
                o["num_workers"] = min(4, ncpu)
            elif o["kind"] == "map":
                o["num_workers"] = ncpu
        vals = []
        for i in range(warmup + steps):
            r = ref.bench_pipeline(primary, g, repeats=1, ids=sample_ids)
            if i >= warmup:
                vals.append(r["items"] / r["cost_time_s"])
        return statistics.median(vals), ncpu, "reference"
    orc = Orc()
    vals = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        for k, smp in enumerate(ref.read_samples(primary, sample_ids)):
            for kind, params, op_id in steps_ops:
                seed = ref.mix_seed(g.get("base_seed", 0), 0, k, op_id)
                impl = ref if kind in REF_OPS and "gather" not in params else orc
                smp = impl.apply_map(kind, params, smp, seed)
        dt = time.perf_counter() - t0
        if i >= warmup:
            vals.append(len(sample_ids) / dt)
    return statistics.median(vals), 1, "port"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="shapenet_part", choices=sorted(CONFIGS))
    ap.add_argument("--quantized", action="store_true", help="LZ4 page variant")
    ap.add_argument("--clouds-per-gpu", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-no-d2h", action="store_true", help="diagnostics: e2e without the batch reads")
    ap.add_argument("--cpu-sample", type=int, default=0, help="clouds per CPU step")
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch size (diagnostics)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    if args.clouds_per_gpu:
        cfg["clouds"] = args.clouds_per_gpu
    rank, world, local = env()
    variant = "quantized (LZ4 pages)" if args.quantized else "raw float (stored-raw pages)"
    config = {"workload": args.config, "desc": cfg["desc"], "variant": variant,
              "clouds_per_gpu_per_step": cfg["clouds"], "points_per_cloud": cfg["points"],
              "batch": cfg["batch"], "group_size": cfg["group"], "slices": SLICES,
              "parallelism": f"record-sharded by slice, {world} independent pipelines",
              "l2": "inputs per step > 126 MB L2 (no flush needed)"}
    metric = "point clouds/sec (PcRecord -> training batch)"
    cpu_sample = args.cpu_sample or {"shapenet_part": 4096, "modelnet40": 64, "kitti": 16,
                                     "s3dis": 2, "scannet": 2}[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        primary = dataset(args.config, cfg, 1, args.quantized, 0, lambda: None)
        g = graph_for(args.config, cfg)
        from paper_2603_16945_b200 import shard
        idx = shard.read_index(primary)
        ids = np.arange(min(cpu_sample, len(idx)), dtype=np.uint64)
        v, ncpu, kind = cpu_reference(primary, g, ids, args.steps, args.warmup)
        line = {"metric": metric, "value": v, "unit": "clouds/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": config,
                "mpoints_per_sec": v * cfg["points"] / 1e6,
                "cpu_baseline": {"value": v, "unit": "clouds/s", "cores": ncpu, "kind": kind,
                                 "sample": f"{len(ids)} clouds per step (first entries); "
                                           f"{'reference Pipeline, ' + str(ncpu) + ' map workers' if kind == 'reference' else 'reference reads/ops + C restatement for App. C ops, 1 thread'}"},
                "e2e": {"value": v, "unit": "clouds/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        if args.config == "shapenet_part":
            line["note"] = "reference downsample ignores the 'gather' extension (seg stays unmoved)"
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        barrier = dist.barrier
    else:
        barrier = lambda: None
    import paper_2603_16945_b200 as P
    from paper_2603_16945_b200 import shard
    primary = dataset(args.config, cfg, world, args.quantized, rank, barrier)
    idx = shard.read_index(primary)
    ids = shard.slice_shard(idx, world, rank)
    g = graph_for(args.config, cfg)
    points_per_step = 0


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
    # roofline of the dominant kernel, measured live with CUDA events on the
    # wave streams (k_cloud and k_page_decode are both timed per wave)
    peak, peak_kind = peaks()
    waves = max(1, st1["waves"] - st0["waves"])
    kern = {}
    for name, ms_key, by_key in (("k_cloud", "cloud_kernel_ms", "cloud_kernel_alg_bytes"),
                                 ("k_page_decode", "decode_kernel_ms", "decode_kernel_alg_bytes")):
        kms = st1[ms_key] - st0[ms_key]
        kby = st1[by_key] - st0[by_key]
        kern[name] = {"ms_per_step": kms / args.steps, "alg_bytes_per_step": kby / args.steps,
                      "achieved_gbs": kby / (kms / 1e3) / 1e9 if kms > 0 else 0.0,
                      "share_of_step": kms / ms if ms else None}
    dom = max(kern, key=lambda k: kern[k]["ms_per_step"])
    # the decode events bracket k_page_decode + k_page_matches (phase 4)
    dram, cap_clouds = ncu_traffic(args.config, "k_page_decode+k_page_matches" if dom == "k_page_decode" else dom)
    alg_per_launch = kern[dom]["alg_bytes_per_step"] * args.steps / waves
    if dram is not None and cap_clouds:  # capture wave -> this run's wave (per-cloud traffic)
        dram = dram / cap_clouds * (clouds_rank / waves)
    achieved = kern[dom]["achieved_gbs"]
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_kind": peak_kind, "traffic": dram,
            "alg_bytes_per_launch": kern[dom]["alg_bytes_per_step"] * args.steps / waves,
            "kernels": kern}
    if dom == "k_page_decode":
        roof["kernel"] = "k_page_decode + k_page_matches"
        roof["note"] = ("latency-bound: one serial LZ4 token/match chain per page "
                        "(DESIGN.md 4.2); HBM fraction reported for completeness")
    if dram is not None and alg_per_launch:
        roof["traffic_over_alg"] = dram / alg_per_launch
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
        v, ncpu, kind = cpu_reference(primary, g, ids_cpu, 1, 0)
        cpu = {"value": v, "unit": "clouds/s", "cores": ncpu, "kind": kind,
               "sample": f"{len(ids_cpu)} clouds of the same dataset; "
                         + (f"reference Pipeline (oracle/_ref), {ncpu} map workers" if kind == "reference"
                            else "reference reads/ops + C restatement for App. C ops, 1 thread")}
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "clouds/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded generators, paper_2603_16945_b200/synth.py)",
                "config": config, "mpoints_per_sec": points_all / (ms_max / 1e3) / 1e6,
                "per_gpu_clouds_per_sec": value / world, "roofline": roof,
                "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
                "gpu_launches": st1["launches"] - st0["launches"],
                "batches_per_step": nb / args.steps}
        if "op_cycles" in st1:  # PCP_OP_TIMING=1 diagnostics: share of k_cloud CTA time
            oc = st1["op_cycles"]
            from paper_2603_16945_b200 import synth
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
