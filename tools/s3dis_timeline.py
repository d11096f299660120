"""S3DIS pipeline run-to-run variance: K pipelines in one process over the
bench dataset (written by a previous bench run), each timing 10 epochs, with
the per-wave timeline (PCP_TIMELINE=1: h0 h1 d0 d1 k0 k1 done host, ms).
python tools/s3dis_timeline.py [runs] [slots]"""
import os
import sys
import time

os.environ["PCP_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2603_16945_b200 as P  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = dict(bench.CONFIGS["s3dis"])
primary = bench.dataset("s3dis", cfg, 1, False, 0, lambda: None)
g = bench.graph_for("s3dis", cfg)
for r in range(runs):
    kw = {"slots": slots} if slots else {}
    p = P.Pipeline(primary, g, epochs=13, **kw)
    n = 0
    t0 = None
    while True:
        b = p.next_batch_raw()
        if b is None:
            break
        n += 1
        if n == 3 * 64:  # after 3 warm-up epochs
            torch.cuda.synchronize()
            t0 = time.perf_counter()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = p.stats()
    p.close()
    tl = st["timeline"]
    print(f"run {r}: {10 * 256 / dt:.0f} rooms/s, slots {st.get('slots', '?')}, waves {len(tl)}")
    for row in tl[-6:]:
        print("   " + " ".join(f"{x:9.1f}" for x in row), f"| k {row[5] - row[4]:.1f} ms")
