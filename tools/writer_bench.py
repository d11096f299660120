"""Writer throughput: host write_dataset (16 threads) vs the device page
encoder, same samples, byte-identical output checked.
  python tools/writer_bench.py [config ...]"""
import json
import os
import shutil
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2603_16945_b200 as P  # noqa: E402

CASES = {"shapenet_part": (4096, False), "shapenet_part_q": (4096, True), "kitti_q": (256, True),
         "kitti": (256, False), "s3dis": (16, False), "s3dis_q": (16, True)}
out = {}
for name in sys.argv[1:] or list(CASES):
    n, q = CASES[name]
    cfg = dict(bench.CONFIGS[name.replace("_q", "")])
    if q and "group_q" in cfg:
        cfg["group"] = cfg["group_q"]
    schema, samples = bench.gen_samples(cfg, n, q)
    raw = sum(sum(v.nbytes for v in s.values() if hasattr(v, "nbytes")) for s in samples)
    res = {}
    for mode in ("host", "device"):
        d = tempfile.mkdtemp()
        P.write_dataset(d, "warm", schema, samples[:4], slice_count=1, group_size=cfg["group"],
                        n_threads=16, device=0 if mode == "device" else None)
        t = time.perf_counter()
        P.write_dataset(d, "ds", schema, samples, slice_count=8, group_size=cfg["group"], n_threads=16,
                        device=0 if mode == "device" else None)
        res[mode] = time.perf_counter() - t
        res[mode + "_dir"] = d
    same = all(open(os.path.join(res["host_dir"], f), "rb").read() == open(os.path.join(res["device_dir"], f), "rb").read()
               for f in os.listdir(res["host_dir"]) if f.startswith("ds."))
    out[name] = {"samples": n, "raw_MB": raw / 1e6, "host_s": res["host"], "device_s": res["device"],
                 "host_MBps": raw / 1e6 / res["host"], "device_MBps": raw / 1e6 / res["device"],
                 "identical": same, "group": cfg["group"]}
    for k in ("host_dir", "device_dir"):
        shutil.rmtree(res[k], ignore_errors=True)
    print(json.dumps({name: out[name]}), flush=True)
