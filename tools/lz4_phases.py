"""LZ4 decode phase clocks (PCP_LZ4_TIMING=1, max over pages) for one
quantized workload: python tools/lz4_phases.py kitti|s3dis|shapenet [n] [group]"""
import os
import sys
import tempfile

os.environ["PCP_LZ4_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16945_b200 as pcp  # noqa: E402
from paper_2603_16945_b200 import synth  # noqa: E402

gen = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
group = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kw = {"mean_points": 1_000_000} if gen == "s3dis" else {}
schema, samples = getattr(synth, gen)(n, quantized=True, **kw)
d = tempfile.mkdtemp()
primary = pcp.write_dataset(d, "ds", schema, samples, slice_count=1, group_size=group)
g = synth.graph(["flip_yz"], batch_size=1)
p = pcp.Pipeline(primary, g)
for _ in p:
    pass
st = p.stats()
p.close()
c = st["lz4_max_phase_cycles"]
print(gen, "pages", n // group, "raw MB/page", round(sum(s["data"].nbytes for s in samples[:group]) / 1e6, 2),
      "max per page: skim (phases 1-2) %.2f ms, phase 3 %.2f ms, warp phase 4 %.2f ms" % tuple(x / 1.965e6 for x in c[:3]),
      "decode_ms", round(st["decode_kernel_ms"], 2), "pj_waves", st["lz4_pj_waves"])
