"""GPU parity of the stateless C-ABI entry points against the compiled
reference: page decode (CRC + CTA-parallel LZ4 + XOR-delta columns), CRC
ranges, and apply_map over cloud sets."""
import ctypes as C
import json
import struct
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(torch, b: bytes, pad=64):
    t = torch.zeros(len(b) + 2 * pad, dtype=torch.uint8, device="cuda")
    if b:
        t[pad:pad + len(b)] = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    return t, pad


def _u64(torch, xs):
    return torch.tensor(list(xs) or [0], dtype=torch.int64, device="cuda")


def _decode_pages(pcp, pages, cols_per_page):
    """pages: serialized EncodedPage bytes; returns [(status, bytes)]."""
    import torch
    blob = b""
    offs = []
    for p in pages:
        offs.append(64 + len(blob))
        blob += p + b"\0" * ((-len(p)) % 16)
    d_bytes, _ = _dev(torch, blob)
    raw_lens = [struct.unpack_from("<Q", p, 1)[0] for p in pages]
    out_off, at = [], 0
    for r in raw_lens:
        out_off.append(at)
        at += r + 64
    d_out = torch.zeros(at + 64, dtype=torch.uint8, device="cuda")
    first, co, cl = [0], [], []
    for cols in cols_per_page:
        for o, l in cols:
            co.append(o)
            cl.append(l)
        first.append(len(co))
    d_po, d_oo = _u64(torch, offs), _u64(torch, out_off)
    d_first = torch.tensor(first, dtype=torch.int32, device="cuda")
    d_co, d_cl = _u64(torch, co), _u64(torch, cl)
    d_st = torch.zeros(len(pages), dtype=torch.int32, device="cuda")
    L = pcp.lib()
    st = L.pcp_decode_pages(C.c_void_p(d_bytes.data_ptr()), C.c_void_p(d_po.data_ptr()), len(pages),
                            C.c_void_p(d_out.data_ptr()), C.c_void_p(d_oo.data_ptr()),
                            C.c_void_p(d_first.data_ptr()), C.c_void_p(d_co.data_ptr()),
                            C.c_void_p(d_cl.data_ptr()), C.c_void_p(d_st.data_ptr()), None)
    assert st == 0, L.pcp_last_error()
    torch.cuda.synchronize()
    out = d_out.cpu().numpy().tobytes()
    res = []
    for i, s in enumerate(d_st.cpu().tolist()):
        res.append((s, out[out_off[i]:out_off[i] + raw_lens[i]]))
    return res


def _ref_decode(ref, page, cols):
    from oracle.ffi import OracleError
    try:
        return 0, ref.decode_page(page, cols)
    except OracleError as e:
        return e.code, None


def _corpus(rng):
    from paper_2603_16945_b200 import synth
    out = [b"", b"\x00" * 5000, rng.integers(0, 256, 3000).astype(np.uint8).tobytes()]
    for n in (13, 100, 4095, 4096, 4097, 70000, 300000):
        out.append(rng.integers(0, 3, n).astype(np.uint8).tobytes())
    walk = np.cumsum(rng.normal(0, 1e-3, 200000)).astype(np.float32)
    out.append(np.round(walk, 3).astype(np.float32).tobytes())
    schema, s = synth.shapenet(3, n_points=2048)
    out.append(b"".join(x["data"].tobytes() + x["seg"].tobytes() for x in s))
    schema, s = synth.kitti(1, lo=60000, hi=60000, quantized=True)
    out.append(s[0]["data"].tobytes() + s[0]["intensity"].tobytes())
    return out


def test_decode_pages_matches_reference(pcp, ref, rng):
    pages, cols = [], []
    for raw in _corpus(rng):
        c = [(0, len(raw) // 8 * 4)] if len(raw) >= 8 else []
        pages.append(ref.encode_page(raw, c))
        cols.append(c)
    got = _decode_pages(pcp, pages, cols)
    for p, c, (st, out) in zip(pages, cols, got):
        rst, rout = _ref_decode(ref, p, c)
        assert st == rst
        assert out == rout


def test_lz4_corruption_verdicts_match_reference(pcp, ref, rng):
    """Mutated LZ4 payloads (CRC re-stamped so decode is reached): the device
    verdict (CorruptPage or bytes) equals lz4::decompress's."""
    from oracle.ffi import OracleError
    raw = rng.integers(0, 256, 2048).astype(np.uint8).tobytes() + b"\x55" * 2048
    raw += rng.integers(0, 4, 9000).astype(np.uint8).tobytes()
    comp = ref.lz4_compress(raw)
    pages, want = [], []
    for k in range(240):
        m = bytearray(comp)
        for _ in range(1 + k % 3):
            m[int(rng.integers(0, len(m)))] ^= int(rng.integers(1, 256))
        if k % 17 == 0:
            m = m[: int(rng.integers(0, len(m)))]
        pay = bytes(m)
        page = struct.pack("<BQQI", 1, len(raw), len(pay), zlib.crc32(pay)) + pay
        pages.append(page)
        try:
            want.append((0, ref.lz4_decompress(pay, len(raw))))
        except OracleError as e:
            want.append((e.code, None))
    got = _decode_pages(pcp, pages, [[]] * len(pages))
    for i, ((gs, go), (ws, wo)) in enumerate(zip(got, want)):
        assert gs == ws, (i, gs, ws)
        if ws == 0:
            assert go == wo, i


def test_crc_ranges(pcp, rng):
    import torch
    data = rng.integers(0, 256, 3_000_000).astype(np.uint8).tobytes()
    d, pad = _dev(torch, data)
    ranges = [(0, 0), (0, 1), (5, 255), (1, 256), (17, 100000), (3, 2_999_990), (123, 2_500_001)]
    d_off = _u64(torch, [pad + a for a, _ in ranges])
    d_len = _u64(torch, [n for _, n in ranges])
    d_crc = torch.zeros(len(ranges), dtype=torch.int32, device="cuda")
    L = pcp.lib()
    assert L.pcp_crc32_ranges(C.c_void_p(d.data_ptr()), C.c_void_p(d_off.data_ptr()),
                              C.c_void_p(d_len.data_ptr()), len(ranges),
                              C.c_void_p(d_crc.data_ptr()), None) == 0
    torch.cuda.synchronize()
    got = [x & 0xFFFFFFFF for x in d_crc.cpu().tolist()]
    assert got == [zlib.crc32(data[a:a + n]) for a, n in ranges]


class _Set(C.Structure):
    _fields_ = [("n_clouds", C.c_uint32), ("d_offset", C.c_void_p), ("d_data", C.c_void_p),
                ("d_normal", C.c_void_p), ("d_color", C.c_void_p), ("d_intensity", C.c_void_p),
                ("d_extra", C.c_void_p * 4), ("extra_elem", C.c_uint32 * 4)]


class _Out(C.Structure):
    _fields_ = [("cap_points", C.c_uint32), ("d_data", C.c_void_p), ("d_normal", C.c_void_p),
                ("d_color", C.c_void_p), ("d_intensity", C.c_void_p), ("d_extra", C.c_void_p * 4),
                ("d_voxel_count", C.c_void_p), ("d_count", C.c_void_p)]


@pytest.mark.parametrize("kind,params", [("normalize", {}), ("translate", {}), ("random_scale", {}),
                                         ("flip_yz", {}), ("color_augment", {}),
                                         ("random_crop", {}), ("downsample", {"num_points": 200}),
                                         ("downsample", {"num_points": 900}),
                                         ("fps", {"num_points": 64}), ("rotate", {}),
                                         ("jitter", {}), ("grid_subsample", {"voxel_size": 0.3}),
                                         ("range_crop", {"lo": [-1, -1, -1], "hi": [1, 0.5, 1]})])
def test_apply_map_cloud_set(pcp, ref, orc, rng, kind, params):
    import torch
    from oracle.ffi import cloud
    sizes = [300, 1, 700, 513]
    clouds = [rng.uniform(-2, 2, (n, 3)).astype(np.float32) for n in sizes]
    normals = [rng.normal(0, 1, (n, 3)).astype(np.float32) for n in sizes]
    colors = [rng.uniform(0, 1, (n, 3)).astype(np.float32) for n in sizes]
    seeds = [int(x) for x in rng.integers(0, 2**63, len(sizes))]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    cap = max(max(sizes), params.get("num_points", 0))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_data, d_nrm, d_col = t(np.concatenate(clouds)), t(np.concatenate(normals)), t(np.concatenate(colors))
    d_off, d_seed = t(off), t(np.array(seeds, dtype=np.uint64).view(np.int64))
    o_data = torch.zeros(len(sizes) * cap * 3, dtype=torch.float32, device="cuda")
    o_nrm, o_col = torch.zeros_like(o_data), torch.zeros_like(o_data)
    o_cnt = torch.zeros(len(sizes), dtype=torch.int32, device="cuda")
    d_st = torch.zeros(len(sizes), dtype=torch.int32, device="cuda")
    s = _Set(len(sizes), d_off.data_ptr(), d_data.data_ptr(), d_nrm.data_ptr(), d_col.data_ptr(), None)
    o = _Out(cap, o_data.data_ptr(), o_nrm.data_ptr(), o_col.data_ptr(), None)
    o.d_count = o_cnt.data_ptr()
    L = pcp.lib()
    L.pcp_apply_map.argtypes = [C.c_int, C.c_char_p, C.POINTER(_Set), C.POINTER(_Out), C.c_void_p,
                                C.c_void_p, C.c_void_p]
    rc = L.pcp_apply_map(pcp.map_kind_from_name(kind), json.dumps(params).encode(), C.byref(s),
                         C.byref(o), d_seed.data_ptr(), d_st.data_ptr(), None)
    assert rc == 0, L.pcp_last_error()
    torch.cuda.synchronize()
    st, cnt = d_st.cpu().numpy(), o_cnt.cpu().numpy()
    od = o_data.cpu().numpy().reshape(len(sizes), cap, 3)
    on = o_nrm.cpu().numpy().reshape(len(sizes), cap, 3)
    oc = o_col.cpu().numpy().reshape(len(sizes), cap, 3)
    tol = kind in ("rotate", "jitter")
    for i in range(len(sizes)):
        smp = {"data": cloud(clouds[i]), "normal": cloud(normals[i]), "color": cloud(colors[i])}
        impl = orc if kind in ("fps", "voxel", "grid_subsample", "range_crop") else ref
        from oracle.ffi import OracleError
        try:
            w = impl.apply_map(kind, params, smp, seeds[i])
        except OracleError as e:
            assert st[i] == e.code, (kind, i, st[i], e.code)
            continue
        assert st[i] == 0
        wd = w["data"].view(np.float32).reshape(-1, 3)
        assert cnt[i] == len(wd)
        for got, name in ((od[i], "data"), (on[i], "normal"), (oc[i], "color")):
            want = w[name].view(np.float32).reshape(-1, 3)
            g = got[: len(want)]
            if tol:
                np.testing.assert_allclose(g, want, rtol=1e-5, atol=1e-6 * max(1, np.abs(want).max()))
            else:
                assert np.array_equal(g.view(np.uint32), want.view(np.uint32)), (kind, i, name)


def _adversarial_fps_pairs(n_pairs, seed=7):
    """Point pairs (P1, P2) whose squared distances to the origin order one way
    with the App. C rounding ((dx*dx + dy*dy) + dz*dz, every op rounded) and
    the other way if the squares were fused into the adds (FMA contraction)."""
    r = np.random.default_rng(seed)
    p = r.uniform(0.5, 1.0, (400000, 3)).astype(np.float32)
    p /= np.linalg.norm(p.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    sq = p * p  # float32, rounded
    unf = (sq[:, 0] + sq[:, 1]) + sq[:, 2]
    p64 = p.astype(np.float64)
    fus = (p64[:, 2] ** 2 + (p64[:, 1] ** 2 + sq[:, 0].astype(np.float64)).astype(np.float32)).astype(np.float32)
    # on the unit sphere the rounded distances take a few ulp-spaced levels;
    # pair a point of a lower level with a point of a higher one whose fused
    # value is not larger
    out = []
    levels = np.unique(unf)
    for lo_v, hi_v in zip(levels[:-1], levels[1:]):
        A = np.flatnonzero(unf == lo_v)
        B = np.flatnonzero(unf == hi_v)
        A = A[np.argsort(-fus[A], kind="stable")]
        B = B[np.argsort(fus[B], kind="stable")]
        for a, b in zip(A, B):
            if fus[a] < fus[b]:
                break
            out.append((p[a], p[b]))
            if len(out) == n_pairs:
                return out
    return out


def _apply_set(pcp, kind, params, clouds, seeds=None):
    import torch
    sizes = [len(c) for c in clouds]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    cap = max(max(sizes), params.get("num_points", 0))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_data, d_off = t(np.concatenate(clouds)), t(off)
    seeds = seeds or [0] * len(clouds)
    d_seed = t(np.array(seeds, dtype=np.uint64).view(np.int64))
    o_data = torch.zeros(len(sizes) * cap * 3, dtype=torch.float32, device="cuda")
    o_cnt = torch.zeros(len(sizes), dtype=torch.int32, device="cuda")
    d_st = torch.zeros(len(sizes), dtype=torch.int32, device="cuda")
    s = _Set(len(sizes), d_off.data_ptr(), d_data.data_ptr(), None, None, None)
    o = _Out(cap, o_data.data_ptr(), None, None, None)
    o.d_count = o_cnt.data_ptr()
    L = pcp.lib()
    L.pcp_apply_map.argtypes = [C.c_int, C.c_char_p, C.POINTER(_Set), C.POINTER(_Out), C.c_void_p,
                                C.c_void_p, C.c_void_p]
    rc = L.pcp_apply_map(pcp.map_kind_from_name(kind), json.dumps(params).encode(), C.byref(s),
                         C.byref(o), d_seed.data_ptr(), d_st.data_ptr(), None)
    assert rc == 0, L.pcp_last_error()
    torch.cuda.synchronize()
    od = o_data.cpu().numpy().reshape(len(sizes), cap, 3)
    return d_st.cpu().numpy(), o_cnt.cpu().numpy(), od


def test_fps_no_fma_contraction(pcp, orc):
    """FPS distances must be computed without FMA (App. C): on these clouds a
    contracted distance picks the other point."""
    from oracle.ffi import cloud
    pairs = _adversarial_fps_pairs(48)
    assert len(pairs) >= 16
    clouds = [np.stack([np.zeros(3, np.float32), a, b]) for a, b in pairs]
    st, cnt, od = _apply_set(pcp, "fps", {"num_points": 2}, clouds)
    for i, c in enumerate(clouds):
        want = orc.apply_map("fps", {"num_points": 2}, {"data": cloud(c)}, 0)["data"]
        want = want.view(np.float32).reshape(-1, 3)
        assert st[i] == 0 and cnt[i] == 2
        assert np.array_equal(want[1], c[2])  # the restatement picks P2 ...
        assert np.array_equal(od[i, :2].view(np.uint32), want.view(np.uint32)), i  # ... and so must we


@pytest.mark.parametrize("n,m", [(3000, 700), (7000, 512), (10000, 1024), (12000, 300), (25000, 900),
                                 (40000, 256), (90000, 64)])
def test_fps_sizes_bit_exact(pcp, orc, rng, n, m):
    """Every FPS path (register P = 8 / 16 / 20, clusters of 2..8 CTAs, and
    the single-CTA global-memory path beyond 8 x 10240 points)
    against the restatement, including duplicated points (exact ties)."""
    from oracle.ffi import cloud
    clouds = []
    for k in range(3):
        c = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
        c[n // 2:n // 2 + 50] = c[:50]  # exact duplicates -> tied distances
        clouds.append(c)
    st, cnt, od = _apply_set(pcp, "fps", {"num_points": m}, clouds)
    for i, c in enumerate(clouds):
        want = orc.apply_map("fps", {"num_points": m}, {"data": cloud(c)}, 0)["data"]
        want = want.view(np.float32).reshape(-1, 3)
        assert st[i] == 0 and cnt[i] == m
        assert np.array_equal(od[i, :m].view(np.uint32), want.view(np.uint32)), i


@pytest.mark.parametrize("vs,extent", [(0.05, 4.0), (1e-5, 20.0)])
def test_voxel_sort_paths(pcp, orc, rng, vs, extent):
    """Voxel/grid through both sorts: packed (key << index bits | index) words
    with 8-bit digits, and the 64-bit key/index fallback when the keys need
    ~21 bits per axis (1e-5 m voxels over 20 m)."""
    from oracle.ffi import cloud
    clouds = [rng.uniform(0, extent, (n, 3)).astype(np.float32) for n in (5000, 777, 1)]
    clouds[0][100:200] = clouds[0][:100]  # duplicates share voxels
    for kind in ("voxel", "grid_subsample"):
        st, cnt, od = _apply_set(pcp, kind, {"voxel_size": vs, "origin": [0, 0, 0]}, clouds)
        for i, c in enumerate(clouds):
            want = orc.apply_map(kind, {"voxel_size": vs, "origin": [0, 0, 0]}, {"data": cloud(c)}, 0)["data"]
            want = want.view(np.float32).reshape(-1, 3)
            assert st[i] == 0 and cnt[i] == len(want), (kind, i)
            assert np.array_equal(od[i, :len(want)].view(np.uint32), want.view(np.uint32)), (kind, i)
