"""Regenerate the golden fixtures in tests/golden/ from the compiled reference
(oracle/_ref/libpcpipe_ref.so, built from the unmodified reference sources by
``make -C oracle reference``).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Outputs (committed, small):
  ops.npz        per reference op: input clouds, seeds, reference outputs
  codec.npz      XOR-delta / LZ4 / page known answers
  ds_raw/, ds_q/ two tiny PcRecord datasets (stored-raw and LZ4 block pages)
  ds_*.npz       reference Pipeline batches for the ShapeNet-part chain
"""
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.ffi import Ref, cloud  # noqa: E402
from paper_2603_16945_b200 import synth  # noqa: E402

OPS = [("normalize", {}), ("translate", {}), ("jitter", {}), ("rotate", {}),
       ("rotate", {"theta": 1.2345}), ("random_scale", {}), ("flip_yz", {}),
       ("color_augment", {}), ("random_crop", {}), ("downsample", {"num_points": 100}),
       ("downsample", {"num_points": 700})]
SEEDS = [1, 12345, 0xDEADBEEFCAFEF00D]
GOLDEN_CHAIN = [("normalize", {}), ("downsample", {"num_points": 256}), ("random_scale", {}),
                ("downsample", {"num_points": 256})]


def clouds():
    rng = np.random.default_rng(20261018)
    out = []
    for n in (1, 2, 7, 300):
        p = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
        c = rng.uniform(0, 1, (n, 3)).astype(np.float32)
        nr = rng.normal(0, 1, (n, 3)).astype(np.float32)
        out.append({"data": cloud(p), "normal": cloud(nr), "color": cloud(c)})
    return out


def main():
    ref = Ref()
    arrays = {}
    cl = clouds()
    for ci, s in enumerate(cl):
        for k in ("data", "normal", "color"):
            arrays[f"in{ci}_{k}"] = s[k]
    for oi, (kind, params) in enumerate(OPS):
        for ci, s in enumerate(cl):
            for si, seed in enumerate(SEEDS):
                o = ref.apply_map(kind, params, s, seed)
                for k in ("data", "normal", "color"):
                    arrays[f"op{oi}_c{ci}_s{si}_{k}"] = o[k]
    arrays["ops_json"] = np.frombuffer(json.dumps(OPS).encode(), np.uint8)
    arrays["seeds"] = np.array(SEEDS, np.uint64)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **arrays)

    rng = np.random.default_rng(7)
    codec = {}
    raw = rng.integers(0, 6, 4096).astype(np.uint8).tobytes()
    codec["lz4_raw"] = np.frombuffer(raw, np.uint8)
    codec["lz4_comp"] = np.frombuffer(ref.lz4_compress(raw), np.uint8)
    walk = np.cumsum(rng.normal(0, 0.01, 3000)).astype(np.float32).tobytes()
    codec["page_raw"] = np.frombuffer(walk, np.uint8)
    cols = [(0, 4000), (4000, 8000)]
    codec["page_cols"] = np.array(cols, np.uint64)
    codec["page_enc"] = np.frombuffer(ref.encode_page(walk, cols), np.uint8)
    codec["crc_123456789"] = np.array([ref.crc32(b"123456789")], np.uint32)
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **codec)

    for name, q in (("ds_raw", False), ("ds_q", True)):
        d = os.path.join(HERE, name)
        shutil.rmtree(d, ignore_errors=True)
        schema, samples = synth.shapenet(24, n_points=512, quantized=q)
        primary = ref.write_dataset(d, "ds", schema, samples, slice_count=2, group_size=8)
        g = synth.graph(GOLDEN_CHAIN, batch_size=4)
        batches = ref.run_pipeline(primary, json.dumps(g))
        out = {"graph": np.frombuffer(json.dumps(g).encode(), np.uint8)}
        for b in batches:
            st = {k: np.concatenate([s[k].view(np.uint8) for s in b["samples"]]) for k in b["samples"][0]}
            for k, v in st.items():
                out[f"b{b['batch_index']}_{k}"] = v
        out["n_batches"] = np.array([len(batches)])
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
