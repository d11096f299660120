"""CPU: pin the C restatement (oracle/liboracle.so) to the reference — the
compiled reference itself (oracle/_ref) and the committed golden fixtures —
plus the reference's own known-answer tests for this path."""
import json
import os
import struct

import numpy as np
import pytest

from oracle.ffi import OracleError, cloud, points

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
REF_OPS = ["normalize", "translate", "jitter", "rotate", "random_scale", "flip_yz",
           "color_augment", "random_crop"]


def _sample(rng, n, with_normal=True, with_color=True, quant=None):
    p = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    if quant:
        p = (np.round(p / quant) * quant).astype(np.float32)
    s = {"data": cloud(p), "label": np.array([3], np.int32)}
    if with_normal:
        s["normal"] = cloud(rng.normal(0, 1, (n, 3)))
    if with_color:
        s["color"] = cloud(rng.uniform(0, 1, (n, 3)))
    return s


# ---------------------------------------------------------------- vs reference
@pytest.mark.parametrize("kind", REF_OPS)
@pytest.mark.parametrize("n", [1, 2, 5, 333, 4096])
def test_restatement_matches_reference_ops(ref, orc, kind, n):
    rng = np.random.default_rng(n)
    s = _sample(rng, n)
    for seed in (0, 7, 123456789, 2**64 - 1):
        a = ref.apply_map(kind, {}, s, seed)
        b = orc.apply_map(kind, {}, s, seed)
        for k in a:
            assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8)), (kind, k, seed)


@pytest.mark.parametrize("t", [1, 100, 999, 1000, 1001, 5000])
def test_restatement_matches_reference_downsample(ref, orc, t):
    rng = np.random.default_rng(t)
    s = _sample(rng, 1000)
    for seed in (3, 99, 2**63 + 5):
        a = ref.apply_map("downsample", {"num_points": t}, s, seed)
        b = orc.apply_map("downsample", {"num_points": t}, s, seed)
        for k in ("data", "normal", "color"):
            assert np.array_equal(a[k], b[k]), (t, k, seed)


def test_normalize_edge_values(ref, orc):
    """tiny coordinates (the exactness certificate's hard case), ±0, big values."""
    rng = np.random.default_rng(5)
    p = rng.uniform(-1, 1, (4000, 3)).astype(np.float32)
    p[::37] *= np.float32(1e-9)
    p[5] = [0.0, -0.0, 3e-38]
    p[6] = [1e20, -1e20, 5.0]
    s = {"data": cloud(p)}
    assert np.array_equal(ref.apply_map("normalize", {}, s, 1)["data"],
                          orc.apply_map("normalize", {}, s, 1)["data"])


def test_crop_and_quantized(ref, orc):
    rng = np.random.default_rng(11)
    for i in range(20):
        s = _sample(rng, 257, quant=0.25)  # many ties on the box boundary
        s["intensity"] = cloud(rng.uniform(0, 1, (257, 1)).repeat(3, 1))[: 257 * 4]
        for seed in range(5):
            a = ref.apply_map("random_crop", {}, s, seed)
            b = orc.apply_map("random_crop", {}, s, seed)
            for k in a:
                assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8)), k


def test_errors_match_reference(ref, orc):
    empty = {"data": np.zeros(0, np.uint8)}
    for kind in REF_OPS:
        with pytest.raises(OracleError) as r:
            ref.apply_map(kind, {}, empty, 1)
        with pytest.raises(OracleError) as o:
            orc.apply_map(kind, {}, empty, 1)
        assert r.value.code == o.value.code == 25  # EmptyCloud
    with pytest.raises(OracleError) as r:
        ref.apply_map("color_augment", {}, {"data": cloud(np.zeros((3, 3)))}, 1)
    assert r.value.code == 24  # MissingField
    with pytest.raises(OracleError) as o:
        orc.apply_map("color_augment", {}, {"data": cloud(np.zeros((3, 3)))}, 1)
    assert o.value.code == 24


def test_mix_seed(ref, orc):
    for args in [(0, 0, 0, 0), (42, 3, 17, 2), (2**64 - 1, 2**63, 12345, 9)]:
        assert ref.mix_seed(*args) == orc.mix_seed(*args)
    # reference test_transforms.cpp:208-217
    seeds = {orc.mix_seed(42, e, i, op) for e in range(4) for i in range(16) for op in range(4)}
    assert len(seeds) == 4 * 16 * 4


def test_lz4_and_pages_vs_reference(ref, orc):
    rng = np.random.default_rng(9)
    for i in range(60):
        n = int(rng.integers(0, 6000))
        raw = rng.integers(0, 4 if i % 2 else 256, n).astype(np.uint8).tobytes()
        comp = ref.lz4_compress(raw)
        assert orc.lz4_decompress(comp, n) == raw
        cols = [(0, n // 8 * 4)] if n >= 8 else []
        page = ref.encode_page(raw, cols)
        assert orc.decode_page(page, cols) == ref.decode_page(page, cols) == raw


def test_lz4_corruption_statuses(ref, orc):
    """test_codec.cpp:72-99: corrupt / truncated streams → CorruptPage."""
    rng = np.random.default_rng(13)
    v = rng.integers(0, 256, 2048).astype(np.uint8).tobytes() + b"\x55" * 2048
    c = ref.lz4_compress(v)
    for cut in (0, len(c) // 4, len(c) - 1):
        for impl in (ref, orc):
            with pytest.raises(OracleError) as e:
                impl.lz4_decompress(c[:cut], len(v))
            assert e.value.code == 7
    for k in range(300):
        m = bytearray(c)
        m[int(rng.integers(0, len(m)))] ^= int(rng.integers(1, 256))
        outs = []
        for impl in (ref, orc):
            try:
                outs.append(impl.lz4_decompress(bytes(m), len(v)))
            except OracleError as e:
                outs.append(e.code)
        assert outs[0] == outs[1]


def test_crc_kats(ref, orc):
    assert orc.crc32(b"123456789") == ref.crc32(b"123456789") == 0xCBF43926
    rng = np.random.default_rng(3)
    for n in (0, 1, 255, 4096, 100001):
        b = rng.integers(0, 256, n).astype(np.uint8).tobytes()
        assert orc.crc32(b) == ref.crc32(b)


def test_checksum_flip_and_truncation(ref, orc):
    """test_format.cpp:185-210."""
    raw = bytes([3]) * 512
    page = bytearray(ref.encode_page(raw, [(0, 512)]))
    page[21 + (len(page) - 21) // 2] ^= 0x10
    for impl in (ref, orc):
        with pytest.raises(OracleError) as e:
            impl.decode_page(bytes(page), [(0, 512)])
        assert e.value.code == 6


# ---------------------------------------------------------------- KATs
def test_xor_delta_known_answers(ref):
    """test_format.cpp:85-104."""
    u = lambda *w: struct.pack(f"<{len(w)}I", *w)
    assert ref.xor_delta(u(0x3F800000), True) == u(0x3F800000)
    assert ref.xor_delta(u(0x3F800000, 0x3F800000), True) == u(0x3F800000, 0)
    assert ref.xor_delta(u(0xDEADBEEF, 0), False) == u(0xDEADBEEF, 0xDEADBEEF)
    assert ref.xor_delta(b"", True) == b""


def test_normalize_known_answers(orc):
    """test_transforms.cpp:37-51."""
    o = points(orc.apply_map("normalize", {}, {"data": cloud([[0, 0, 0], [2, 0, 0]])}, 1)["data"])
    assert o.tolist() == [[-1, 0, 0], [1, 0, 0]]
    o = points(orc.apply_map("normalize", {}, {"data": cloud([[3, 3, 3]] * 3)}, 1)["data"])
    assert (o == 0).all()


def test_rotate_normal_known_answer(orc):
    """test_transforms.cpp:78-86: theta = pi/2 maps normal (1,0,0) → (0,1,0)."""
    s = {"data": cloud([[1, 0, 0]]), "normal": cloud([[1, 0, 0]])}
    o = points(orc.apply_map("rotate", {"theta": np.pi / 2}, s, 1)["normal"])
    assert abs(o[0, 0]) < 1e-6 and abs(o[0, 1] - 1) < 1e-6 and o[0, 2] == 0


# ---------------------------------------------------------------- App. C ops
def test_fps_known_answer(orc):
    """Line of points: FPS from index 0 picks the far end, then the middle."""
    p = np.zeros((11, 3), np.float32)
    p[:, 0] = np.arange(11)
    o = points(orc.apply_map("fps", {"num_points": 3}, {"data": cloud(p)}, 0)["data"])
    assert o[:, 0].tolist() == [0, 10, 5]
    # ties → lowest index; duplicates keep mind 0
    p = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [1, 0, 0]], np.float32)
    o = points(orc.apply_map("fps", {"num_points": 3}, {"data": cloud(p)}, 0)["data"])
    assert o[:, 0].tolist() == [0, 1, -1]
    with pytest.raises(OracleError):
        orc.apply_map("fps", {"num_points": 5}, {"data": cloud(p)}, 0)


def test_range_crop_known_answer(orc):
    p = np.array([[0, 0, 0], [5, 0, 0], [1, 1, 1], [-1, 0, 0]], np.float32)
    s = {"data": cloud(p), "intensity": np.arange(4, dtype=np.float32).view(np.uint8)}
    o = orc.apply_map("range_crop", {"lo": [0, 0, 0], "hi": [1, 1, 1]}, s, 0)
    assert points(o["data"]).tolist() == [[0, 0, 0], [1, 1, 1]]
    assert o["intensity"].view(np.float32).tolist() == [0.0, 2.0]


# ---------------------------------------------------------------- golden fixtures
def test_golden_ops(orc):
    g = np.load(os.path.join(GOLD, "ops.npz"))
    ops = json.loads(bytes(g["ops_json"]).decode())
    seeds = [int(x) for x in g["seeds"]]
    for oi, (kind, params) in enumerate(ops):
        for ci in range(4):
            s = {k: g[f"in{ci}_{k}"] for k in ("data", "normal", "color")}
            for si, seed in enumerate(seeds):
                o = orc.apply_map(kind, params, s, seed)
                for k in ("data", "normal", "color"):
                    assert np.array_equal(o[k], g[f"op{oi}_c{ci}_s{si}_{k}"]), (kind, ci, si, k)


def test_golden_codec(orc):
    g = np.load(os.path.join(GOLD, "codec.npz"))
    assert orc.lz4_decompress(g["lz4_comp"].tobytes(), g["lz4_raw"].size) == g["lz4_raw"].tobytes()
    cols = [tuple(int(x) for x in c) for c in g["page_cols"]]
    assert orc.decode_page(g["page_enc"].tobytes(), cols) == g["page_raw"].tobytes()
    assert orc.crc32(b"123456789") == int(g["crc_123456789"][0])
