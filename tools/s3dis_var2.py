"""bench.py's timed() structure in one process: warm-up pipeline (3 epochs),
then a fresh 10-epoch pipeline timed from its first batch request with CUDA
events, with / without the NVML clock sampler.  python tools/s3dis_var2.py [runs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2603_16945_b200 as P  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = dict(bench.CONFIGS["s3dis"])
primary = bench.dataset("s3dis", cfg, 1, False, 0, lambda: None)
g = bench.graph_for("s3dis", cfg)


def timed(steps, clocks):
    p = P.Pipeline(primary, g, epochs=steps)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ck = bench.Clocks(0) if clocks else None
    if ck:
        ck.__enter__()
    e0.record()
    while p.next_batch_raw() is not None:
        pass
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    if ck:
        ck.__exit__(None, None, None)
    p.close()
    return e0.elapsed_time(e1) / steps


for r in range(runs):
    for clocks in (True, False):
        timed(3, False)
        ms = timed(10, clocks)
        print(f"run {r} clocks={clocks}: {256 / ms * 1e3:.0f} rooms/s ({ms:.1f} ms/step)", flush=True)
