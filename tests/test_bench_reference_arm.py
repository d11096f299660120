"""bench.py --impl reference: the reference arm runs the reference CPU
pipeline (oracle/_ref) on pages written by the reference's own writer and
maps no library of this repo (the product .so must not be loaded)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,sample", [("shapenet_part", 128), ("kitti", 8)])
def test_reference_arm_line(config, sample):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", config, "--steps", "1", "--warmup", "0",
                          "--cpu-sample", str(sample)],
                         capture_output=True, text=True, timeout=600, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["mapped_repo_libraries"] == []
    assert line["cpu_baseline"]["kind"] == ("reference" if config == "shapenet_part" else "port")
    assert line["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
    assert line["e2e"]["h2d_bytes_per_step"] == 0
