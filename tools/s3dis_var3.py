"""Fresh-pipeline S3DIS timing (bench.py's timed() structure) under several
slot counts, alternating, in one process: python tools/s3dis_var3.py runs slots..."""
import os
import sys

os.environ["PCP_TIMELINE"] = "1"

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2603_16945_b200 as P  # noqa: E402

runs = int(sys.argv[1])
slot_list = [int(x) for x in sys.argv[2:]]
cfg = dict(bench.CONFIGS["s3dis"])
primary = bench.dataset("s3dis", cfg, 1, False, 0, lambda: None)
g = bench.graph_for("s3dis", cfg)


def timed(steps, slots):
    p = P.Pipeline(primary, g, epochs=steps, slots=slots)
    torch.cuda.synchronize()
    if os.environ.get("SPIN_MS"):  # keep the GPU busy right before the timed region (clock ramp test)
        x = torch.randn(8192, 8192, device="cuda")
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        while True:
            x = x @ x
            x = x / x.norm()
            s1.record()
            s1.synchronize()
            if s0.elapsed_time(s1) > float(os.environ["SPIN_MS"]):
                break
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while p.next_batch_raw() is not None:
        pass
    e1.record()
    e1.synchronize()
    tl = p.stats()["timeline"]
    p.close()
    ms = e0.elapsed_time(e1) / steps
    if steps > 3:
        t0 = tl[0][2]
        print(f"  {256 / ms * 1e3:.0f}/s  waves (d0, k0, k1, done, host) rel ms: " +
              "; ".join(f"{r[2]-t0:.0f},{r[4]-t0:.0f},{r[5]-t0:.0f},{r[6]-t0:.0f},{r[7]-t0:.0f}" for r in tl), flush=True)
    return ms


res = {s: [] for s in slot_list}
for r in range(runs):
    for s in slot_list:
        timed(3, s)
        res[s].append(round(256 / timed(10, s) * 1e3))
for s in slot_list:
    print(f"slots {s}: {res[s]}", flush=True)
