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
pinned host memory, per-wave H2D and per-batch D2H of every field inside the
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
                  desc="KITTI-shaped ~120k-pt XYZI frames: range crop, rotate, flip_yz; B 4"),
    "s3dis": dict(gen="s3dis", kw={"mean_points": 1_000_000}, clouds=64, group=1, batch=4,
                  points=1_000_000, desc="S3DIS-shaped ~1M-pt XYZRGB rooms: random_crop, "
                  "downsample 4096; B 4"),
}
CHAIN_OF = {"shapenet_part": "shapenet_part", "modelnet40": "modelnet40", "kitti": "kitti",
            "s3dis": "s3dis"}
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
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev, self.rows, self.p = dev, [], None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic(workload):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        k = s.get(workload, {}).get("k_cloud", {})
        return k.get("dram_bytes_per_launch"), k.get("alg_bytes_per_launch")
    except (OSError, ValueError):
        return None, None


def graph_for(cfg_name, cfg, workers=1):
    from paper_2603_16945_b200 import synth
    return synth.graph(synth.CHAINS[CHAIN_OF[cfg_name]], batch_size=cfg["batch"], base_seed=42,
                       workers=workers)


def cpu_reference(primary, graph, sample_ids, steps, warmup):
    """The reference Pipeline (oracle/_ref: unmodified reference sources)
    with all host threads, run_benchmark-style timing (bench.cpp:43-96)."""
    from oracle.ffi import Ref
    ref = Ref()
    ncpu = os.cpu_count() or 1
    g = json.loads(json.dumps(graph))
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
    return statistics.median(vals), ncpu, g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="shapenet_part", choices=sorted(CONFIGS))
    ap.add_argument("--quantized", action="store_true", help="LZ4 page variant")
    ap.add_argument("--clouds-per-gpu", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="clouds per CPU step")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
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
    cpu_sample = args.cpu_sample or {"shapenet_part": 4096, "modelnet40": 512, "kitti": 32,
                                     "s3dis": 4}[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        primary = dataset(args.config, cfg, 1, args.quantized, 0, lambda: None)
        g = graph_for(args.config, cfg)
        from paper_2603_16945_b200 import shard
        idx = shard.read_index(primary)
        ids = np.arange(min(cpu_sample, len(idx)), dtype=np.uint64)
        v, ncpu, _ = cpu_reference(primary, g, ids, args.steps, args.warmup)
        line = {"metric": metric, "value": v, "unit": "clouds/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": config,
                "mpoints_per_sec": v * cfg["points"] / 1e6,
                "cpu_baseline": {"value": v, "unit": "clouds/s", "cores": ncpu, "kind": "reference",
                                 "sample": f"{len(ids)} clouds per step (first entries), reference "
                                           f"Pipeline, {ncpu} map workers"},
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
        p = P.Pipeline(primary, g, ids=ids, device=local, epochs=steps, resident=resident)
        st0 = p.stats()
        pinned = {}
        d2h_bytes = 0
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(local) as ck:
            e0.record()
            nb = 0
            for b in p:
                nb += 1
                if d2h:
                    for name, (kind, ptr, nbytes, offs, uni) in b.fields.items():
                        if name not in pinned or pinned[name].numel() < nbytes:
                            pinned[name] = torch.empty(max(nbytes, 1), dtype=torch.uint8,
                                                       pin_memory=True)
                        P.lib().pcp_memcpy_d2h(pinned[name].data_ptr(), ptr, nbytes, b.stream)
                        d2h_bytes += nbytes
            torch.cuda.synchronize()
            e1.record()
            e1.synchronize()
        ms = e0.elapsed_time(e1)
        st1 = p.stats()
        p.close()
        return ms, st0, st1, nb, d2h_bytes, ck.summary()

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
    # roofline of the dominant kernel (k_cloud), measured live with CUDA events
    kms = st1["cloud_kernel_ms"] - st0["cloud_kernel_ms"]
    kbytes = st1["cloud_kernel_alg_bytes"] - st0["cloud_kernel_alg_bytes"]
    waves = max(1, st1["waves"] - st0["waves"] + 1)
    peak, peak_kind = peaks()
    achieved = kbytes / (kms / 1e3) / 1e9 if kms > 0 else 0.0
    dram, alg_per_launch = ncu_traffic(args.config)
    roof = {"bound": "hbm", "kernel": "k_cloud", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "peak_kind": peak_kind,
            "traffic": dram, "alg_bytes_per_launch": kbytes / waves,
            "kernel_ms_per_step": kms / args.steps,
            "kernel_share_of_step": kms / ms if ms else None,
            "step_hbm_gbs": kbytes / (ms / 1e3) / 1e9}
    if dram is not None and alg_per_launch:
        roof["traffic_over_alg"] = dram / alg_per_launch
    e2e = None
    if not args.no_e2e:
        ems, est0, est1, enb, d2h, _ = timed(False, args.steps, True)
        te = torch.tensor([ems], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_clouds = est1["clouds"] - est0["clouds"]
        tc = torch.tensor([e_clouds], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tc)
        e2e = {"value": float(tc.item()) / (float(te.item()) / 1e3), "unit": "clouds/s",
               "h2d_bytes_per_step": (est1["h2d_bytes"] - est0["h2d_bytes"]) // args.steps,
               "d2h_bytes_per_step": d2h // args.steps,
               "path": "pcp_pipeline_open(resident=false) + pcp_pipeline_next_batch + "
                       "pcp_memcpy_d2h of every batch field into pinned host memory"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ids_cpu = np.arange(min(cpu_sample, len(idx)), dtype=np.uint64)
        v, ncpu, _ = cpu_reference(primary, g, ids_cpu, 1, 0)
        cpu = {"value": v, "unit": "clouds/s", "cores": ncpu, "kind": "reference",
               "sample": f"{len(ids_cpu)} clouds of the same dataset, reference Pipeline "
                         f"(oracle/_ref), {ncpu} map workers"}
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
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
