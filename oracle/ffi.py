"""oracle/ffi.py — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU oracles:

* ``Ref``  — oracle/_ref/libpcpipe_ref.so: the unmodified reference sources
  (/root/reference/proj/core/src) + oracle/ref_shim.cpp.  The strongest oracle:
  its outputs ARE the reference's outputs.
* ``Orc``  — oracle/liboracle.so: the plain-C restatement (pcpipe_oracle.c),
  pinned against ``Ref`` in tests/test_oracle.py, and the only oracle for the
  ops the reference lacks (fps / voxel / range_crop).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.

Samples are ``dict[str, np.ndarray]``: bytes fields are ``uint8`` arrays (a
float32 ``[N,3]`` cloud is its 12N raw bytes), int32/int64/float32/float64
fields are arrays of that dtype, strings are ``str``.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpcpipe_ref.so")
ORC_SO = os.path.join(HERE, "liboracle.so")

_KIND_OF_DTYPE = {np.dtype(np.uint8): 0, np.dtype(np.int32): 1, np.dtype(np.int64): 2,
                  np.dtype(np.float32): 3, np.dtype(np.float64): 4}
_DTYPE_OF_KIND = {0: np.uint8, 1: np.int32, 2: np.int64, 3: np.float32, 4: np.float64}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


# --------------------------------------------------------------------------- TLV
def encode_sample(s: dict) -> bytes:
    out = [struct.pack("<I", len(s))]
    for name in sorted(s):  # std::map order
        v = s[name]
        nb = name.encode()
        if isinstance(v, str):
            kind, raw = 5, v.encode()
        else:
            a = np.ascontiguousarray(v)
            kind, raw = _KIND_OF_DTYPE[a.dtype], a.tobytes()
        out.append(struct.pack("<H", len(nb)) + nb + struct.pack("<BQ", kind, len(raw)) + raw)
    return b"".join(out)


def _decode_sample(buf: bytes, pos: int):
    (nf,) = struct.unpack_from("<I", buf, pos)
    pos += 4
    s = {}
    for _ in range(nf):
        (nl,) = struct.unpack_from("<H", buf, pos)
        pos += 2
        name = buf[pos:pos + nl].decode()
        pos += nl
        kind, nbytes = struct.unpack_from("<BQ", buf, pos)
        pos += 9
        raw = buf[pos:pos + nbytes]
        pos += nbytes
        s[name] = raw.decode() if kind == 5 else np.frombuffer(raw, dtype=_DTYPE_OF_KIND[kind]).copy()
    return s, pos


def decode_sample(buf: bytes) -> dict:
    return _decode_sample(buf, 0)[0]


def decode_samples(buf: bytes) -> list:
    (n,) = struct.unpack_from("<I", buf, 0)
    pos, out = 4, []
    for _ in range(n):
        s, pos = _decode_sample(buf, pos)
        out.append(s)
    return out


def decode_batches(buf: bytes) -> list:
    (n,) = struct.unpack_from("<I", buf, 0)
    pos, out = 4, []
    for _ in range(n):
        epoch, bidx, ns = struct.unpack_from("<QQI", buf, pos)
        pos += 20
        samples = []
        for _ in range(ns):
            s, pos = _decode_sample(buf, pos)
            samples.append(s)
        out.append({"epoch": epoch, "batch_index": bidx, "samples": samples})
    return out


def stacked(samples: list) -> dict:
    """Batch::stacked (pipeline.cpp:170-200): per-field concatenation."""
    out = {}
    for name, v0 in samples[0].items():
        if isinstance(v0, str):
            raise OracleError(8, "string fields cannot be stacked")
        for s in samples[1:]:
            if s[name].shape != v0.shape:
                raise OracleError(8, f"ragged field '{name}'")
        out[name] = np.concatenate([s[name] for s in samples])
    return out


# --------------------------------------------------------------------------- Ref
class Ref:
    """The compiled reference (oracle/_ref/libpcpipe_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle reference)")
        L = self.L = C.CDLL(path)
        u8p, u64p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)
        self._outp = (C.POINTER(C.c_uint8), C.c_size_t)
        L.ref_last_error.restype = C.c_char_p
        L.ref_crc32.restype = C.c_uint32
        L.ref_crc32.argtypes = [C.c_char_p, C.c_size_t]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64] * 4
        L.ref_lz4_compress.restype = C.c_size_t
        L.ref_lz4_compress.argtypes = [C.c_char_p, C.c_size_t, u8p, C.c_size_t]
        L.ref_lz4_decompress.argtypes = [C.c_char_p, C.c_size_t, u8p, C.c_size_t]
        L.ref_xor_delta.argtypes = [C.c_int, C.c_char_p, C.c_size_t, C.c_uint32,
                                    C.POINTER(u8p), C.POINTER(C.c_size_t)]
        L.ref_encode_block_page.argtypes = [C.c_char_p, C.c_size_t, u64p, u64p, C.c_size_t,
                                            C.c_int, C.POINTER(u8p), C.POINTER(C.c_size_t)]
        L.ref_decode_block_page.argtypes = [C.c_char_p, C.c_size_t, u64p, u64p, C.c_size_t,
                                            C.POINTER(u8p), C.POINTER(C.c_size_t)]
        L.ref_apply_map.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t, C.c_uint64,
                                    C.POINTER(u8p), C.POINTER(C.c_size_t)]
        L.ref_write_dataset.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                        C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32]
        L.ref_read_samples.argtypes = [C.c_char_p, u64p, C.c_size_t, C.POINTER(u8p),
                                       C.POINTER(C.c_size_t)]
        L.ref_index_json.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.POINTER(u8p),
                                     C.POINTER(C.c_size_t)]
        L.ref_run_pipeline.argtypes = [C.c_char_p, C.c_char_p, u64p, C.c_size_t, C.c_uint64,
                                       C.POINTER(u8p), C.POINTER(C.c_size_t)]
        L.ref_bench_pipeline.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, u64p, C.c_size_t,
                                         C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.ref_bench_composed.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint32, u64p,
                                         C.c_size_t, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.ref_simulate_dp.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, C.c_uint32,
                                      C.POINTER(C.c_double), C.c_size_t, C.c_double,
                                      C.POINTER(C.c_double)]
        L.ref_free.argtypes = [C.c_void_p]

    def _check(self, st):
        if st:
            raise OracleError(st, self.L.ref_last_error().decode())

    def _call_out(self, fn, *args) -> bytes:
        p = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        self._check(fn(*args, C.byref(p), C.byref(n)))
        try:
            return C.string_at(p, n.value)
        finally:
            self.L.ref_free(p)

    @staticmethod
    def _u64(a):
        if a is None:
            return None, 0
        arr = np.ascontiguousarray(a, dtype=np.uint64)
        return arr.ctypes.data_as(C.POINTER(C.c_uint64)), len(arr), arr

    # codec
    def crc32(self, b: bytes) -> int:
        return self.L.ref_crc32(b, len(b))

    def mix_seed(self, base, epoch, index, op) -> int:
        return self.L.ref_mix_seed(base, epoch, index, op)

    def lz4_compress(self, b: bytes) -> bytes:
        cap = len(b) + len(b) // 255 + 16
        out = (C.c_uint8 * cap)()
        k = self.L.ref_lz4_compress(b, len(b), out, cap)
        if k == 0:
            raise OracleError(7, "lz4 compress overflow")
        return bytes(out[:k])

    def lz4_decompress(self, b: bytes, raw_len: int) -> bytes:
        out = (C.c_uint8 * max(raw_len, 1))()
        self._check(self.L.ref_lz4_decompress(b, len(b), out, raw_len))
        return bytes(out[:raw_len])

    def xor_delta(self, b: bytes, encode: bool, width: int = 4) -> bytes:
        return self._call_out(self.L.ref_xor_delta, int(encode), b, len(b), width)

    def _cols(self, cols):
        off = np.array([c[0] for c in cols] or [0], dtype=np.uint64)
        ln = np.array([c[1] for c in cols] or [0], dtype=np.uint64)
        return off, ln

    def encode_page(self, raw: bytes, cols=(), scalar=False) -> bytes:
        off, ln = self._cols(cols)
        return self._call_out(self.L.ref_encode_block_page, raw, len(raw),
                              off.ctypes.data_as(C.POINTER(C.c_uint64)),
                              ln.ctypes.data_as(C.POINTER(C.c_uint64)), len(cols), int(scalar))

    def decode_page(self, page: bytes, cols=()) -> bytes:
        off, ln = self._cols(cols)
        return self._call_out(self.L.ref_decode_block_page, page, len(page),
                              off.ctypes.data_as(C.POINTER(C.c_uint64)),
                              ln.ctypes.data_as(C.POINTER(C.c_uint64)), len(cols))

    # operators
    def apply_map(self, kind: str, params: dict | None, sample: dict, seed: int) -> dict:
        tlv = encode_sample(sample)
        out = self._call_out(self.L.ref_apply_map, kind.encode(),
                             json.dumps(params or {}).encode(), tlv, len(tlv), seed)
        return decode_sample(out)

    # dataset
    def write_dataset(self, out_dir, stem, schema: dict, samples: list, slice_count=1,
                      group_size=256):
        tlv = b"".join(encode_sample(s) for s in samples)
        self._check(self.L.ref_write_dataset(str(out_dir).encode(), stem.encode(),
                                             json.dumps(schema).encode(), tlv, len(tlv),
                                             len(samples), slice_count, group_size))
        return os.path.join(str(out_dir), stem + ".pcrecord")

    def read_samples(self, primary, ids) -> list:
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        out = self._call_out(self.L.ref_read_samples, str(primary).encode(),
                             ids.ctypes.data_as(C.POINTER(C.c_uint64)), len(ids))
        return decode_samples(out)

    def index(self, primary, num_shards=0, shard_id=0) -> dict:
        out = self._call_out(self.L.ref_index_json, str(primary).encode(), num_shards, shard_id)
        return json.loads(out.decode())

    def run_pipeline(self, primary, graph: dict | str, ids=None, epochs=1) -> list:
        g = graph if isinstance(graph, str) else json.dumps(graph)
        if ids is None:
            p, n = None, 0
        else:
            arr = np.ascontiguousarray(ids, dtype=np.uint64)
            p, n = arr.ctypes.data_as(C.POINTER(C.c_uint64)), len(arr)
        out = self._call_out(self.L.ref_run_pipeline, str(primary).encode(), g.encode(), p, n,
                             epochs)
        return decode_batches(out)

    def bench_pipeline(self, primary, graph: dict | str, repeats=1, ids=None) -> dict:
        g = graph if isinstance(graph, str) else json.dumps(graph)
        if ids is None:
            p, n = None, 0
        else:
            arr = np.ascontiguousarray(ids, dtype=np.uint64)
            p, n = arr.ctypes.data_as(C.POINTER(C.c_uint64)), len(arr)
        t, items, batches, cpu = C.c_double(), C.c_uint64(), C.c_uint64(), C.c_double()
        self._check(self.L.ref_bench_pipeline(str(primary).encode(), g.encode(), repeats, p, n,
                                              C.byref(t), C.byref(items), C.byref(batches),
                                              C.byref(cpu)))
        return {"cost_time_s": t.value, "items": items.value, "batches": batches.value,
                "avg_cpu_percent": cpu.value}


    def bench_composed(self, primary, graph: dict, prefix: list, repeats=1, ids=None) -> dict:
        """run_benchmark over the reference Pipeline whose SourceFn applies
        ``prefix`` ([{"map", "params", "op_id"}], App. C ops via the C
        restatement, reference ops via the reference apply_map) after
        read_sample; ``graph`` carries the reference-op suffix."""
        arr = np.ascontiguousarray(ids if ids is not None else [], dtype=np.uint64)
        p = arr.ctypes.data_as(C.POINTER(C.c_uint64)) if ids is not None else None
        t, items, batches, cpu = C.c_double(), C.c_uint64(), C.c_uint64(), C.c_double()
        self._check(self.L.ref_bench_composed(str(primary).encode(), json.dumps(graph).encode(),
                                              json.dumps(prefix).encode(), repeats, p,
                                              len(arr) if ids is not None else 0,
                                              C.byref(t), C.byref(items), C.byref(batches),
                                              C.byref(cpu)))
        return {"cost_time_s": t.value, "items": items.value, "batches": batches.value,
                "avg_cpu_percent": cpu.value}


    def simulate_dp(self, primary, num_devices, epochs, per_device_batch, params, lr):
        """simulate_data_parallel (distributed.cpp:88-164): final params, max divergence."""
        p = (C.c_double * len(params))(*params)
        div = C.c_double()
        self._check(self.L.ref_simulate_dp(str(primary).encode(), num_devices, epochs, per_device_batch,
                                           p, len(params), lr, C.byref(div)))
        return list(p), div.value


# --------------------------------------------------------------------------- Orc
class _Params(C.Structure):
    _fields_ = [("has_theta", C.c_int), ("theta", C.c_float), ("num_points", C.c_int64),
                ("gather_intensity", C.c_int), ("gather_extra", C.c_int),
                ("voxel_size", C.c_float), ("has_origin", C.c_int), ("origin", C.c_float * 3),
                ("lo", C.c_float * 3), ("hi", C.c_float * 3)]


_FP = C.POINTER(C.c_float)


class _Cloud(C.Structure):
    _fields_ = [("data", _FP), ("normal", _FP), ("color", _FP), ("intensity", _FP),
                ("n", C.c_size_t), ("n_normal", C.c_size_t), ("n_color", C.c_size_t),
                ("n_intensity", C.c_size_t), ("extra", C.POINTER(C.c_uint8) * 4),
                ("extra_elem", C.c_size_t * 4), ("n_extra", C.c_size_t * 4),
                ("counts", C.POINTER(C.c_int32)), ("n_counts", C.c_size_t), ("cap", C.c_size_t)]


ORC_KINDS = {"normalize": 0, "translate": 1, "jitter": 2, "rotate": 3, "random_scale": 4,
             "flip_yz": 5, "color_augment": 6, "random_crop": 7, "downsample": 8,
             "fps": 16, "voxel": 17, "grid_subsample": 17, "range_crop": 18}
_POINT3 = ("data", "normal", "color")


class Orc:
    """The plain-C restatement (oracle/liboracle.so)."""

    def __init__(self, path: str = ORC_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle restatement)")
        L = self.L = C.CDLL(path)
        L.orc_crc32.restype = C.c_uint32
        L.orc_crc32.argtypes = [C.c_char_p, C.c_size_t]
        L.orc_lz4_decompress.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_uint8), C.c_size_t]
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_mix_seed.argtypes = [C.c_uint64] * 4
        L.orc_apply_map.argtypes = [C.c_int, C.POINTER(_Params), C.POINTER(_Cloud), C.c_uint64]
        L.orc_decode_page.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_uint8),
                                      C.c_size_t, C.POINTER(C.c_size_t)]

    def crc32(self, b: bytes) -> int:
        return self.L.orc_crc32(b, len(b))

    def mix_seed(self, base, epoch, index, op) -> int:
        return self.L.orc_mix_seed(base, epoch, index, op)

    def lz4_decompress(self, b: bytes, raw_len: int) -> bytes:
        out = (C.c_uint8 * max(raw_len, 1))()
        st = self.L.orc_lz4_decompress(b, len(b), out, raw_len)
        if st:
            raise OracleError(st, "lz4")
        return bytes(out[:raw_len])

    def decode_page(self, page: bytes, cols=()) -> bytes:
        off = np.array([c[0] for c in cols] or [0], dtype=np.uint64)
        ln = np.array([c[1] for c in cols] or [0], dtype=np.uint64)
        (raw_len,) = struct.unpack_from("<Q", page, 1)
        out = (C.c_uint8 * max(raw_len, 1))()
        n = C.c_size_t()
        st = self.L.orc_decode_page(page, len(page), off.ctypes.data_as(C.POINTER(C.c_uint64)),
                                    ln.ctypes.data_as(C.POINTER(C.c_uint64)), len(cols), out,
                                    raw_len, C.byref(n))
        if st:
            raise OracleError(st, "decode_page")
        return bytes(out[:n.value])

    def apply_map(self, kind: str, params: dict | None, sample: dict, seed: int,
                  gather: tuple = ()) -> dict:
        """apply_map restatement.  ``gather`` names extra per-point bytes fields
        (e.g. "seg") that index ops move with the points (App. C extension);
        params["gather"] is honoured the same way."""
        params = dict(params or {})
        gather = tuple(gather) + tuple(params.get("gather", ()))
        if kind not in ORC_KINDS:
            raise OracleError(26, f"unknown map '{kind}'")
        s = dict(sample)
        if "data" not in s or isinstance(s["data"], str) or s["data"].dtype != np.uint8:
            raise OracleError(24, "sample has no 'data' coordinates")
        f3 = {}
        for name in _POINT3:
            v = s.get(name)
            if v is None or isinstance(v, str) or v.dtype != np.uint8 or (name != "data" and v.size == 0):
                continue
            if v.size % 12:
                raise OracleError(24, f"{name} is not an Nx3 float32 blob")
            f3[name] = v.view(np.float32).reshape(-1, 3)
        n = len(f3["data"])
        if n == 0:
            raise OracleError(25, "zero points")
        tgt = int(params.get("num_points", 0))
        cap = max(n, tgt, max((len(a) for a in f3.values()), default=0), 1)
        cl = _Cloud()
        keep = []

        def buf3(name):
            a = np.zeros((cap, 3), np.float32)
            a[:len(f3[name])] = f3[name]
            keep.append(a)
            return a

        bufs = {}
        for name in f3:
            bufs[name] = buf3(name)
            setattr(cl, name, bufs[name].ctypes.data_as(_FP))
        cl.n = n
        cl.n_normal = len(f3["normal"]) if "normal" in f3 else 0
        cl.n_color = len(f3["color"]) if "color" in f3 else 0
        inten = s.get("intensity")
        if inten is not None and not isinstance(inten, str) and inten.dtype == np.uint8 and inten.size:
            iv = inten[: inten.size // 4 * 4].view(np.float32)
            bi = np.zeros(max(cap, len(iv)), np.float32)
            bi[:len(iv)] = iv
            keep.append(bi)
            bufs["intensity"] = bi
            cl.intensity = bi.ctypes.data_as(_FP)
            cl.n_intensity = len(iv)
        extra_names = [g for g in gather if g in s and g != "intensity"]
        for e, name in enumerate(extra_names[:4]):
            raw = s[name]
            es = raw.size // n if n else 1
            b = np.zeros(cap * es, np.uint8)
            b[:raw.size] = raw
            keep.append(b)
            bufs[name] = b
            cl.extra[e] = b.ctypes.data_as(C.POINTER(C.c_uint8))
            cl.extra_elem[e] = es
            cl.n_extra[e] = raw.size // es
        counts = None
        if kind in ("voxel", "grid_subsample") and params.get("counts", kind == "voxel"):
            counts = np.zeros(cap, np.int32)
            cl.counts = counts.ctypes.data_as(C.POINTER(C.c_int32))
        cl.cap = cap
        p = _Params()
        if "theta" in params:
            p.has_theta, p.theta = 1, float(np.float32(params["theta"]))
        p.num_points = tgt
        p.gather_intensity = int("intensity" in gather)
        p.gather_extra = int(bool(extra_names))
        p.voxel_size = float(params.get("voxel_size", 0.0))
        if "origin" in params:
            p.has_origin = 1
            p.origin[:] = [float(x) for x in params["origin"]]
        if "lo" in params:
            p.lo[:] = [float(x) for x in params["lo"]]
            p.hi[:] = [float(x) for x in params["hi"]]
        st = self.L.orc_apply_map(ORC_KINDS[kind], C.byref(p), C.byref(cl), seed)
        if st:
            raise OracleError(st, f"apply_map({kind})")
        out = dict(s)
        out["data"] = np.ascontiguousarray(bufs["data"][:cl.n]).view(np.uint8).reshape(-1)
        if "normal" in f3:
            out["normal"] = np.ascontiguousarray(bufs["normal"][:cl.n_normal]).view(np.uint8).reshape(-1)
        if "color" in f3:
            out["color"] = np.ascontiguousarray(bufs["color"][:cl.n_color]).view(np.uint8).reshape(-1)
        if "intensity" in bufs:
            out["intensity"] = np.ascontiguousarray(bufs["intensity"][:cl.n_intensity]).view(np.uint8).reshape(-1)
        for e, name in enumerate(extra_names[:4]):
            out[name] = bufs[name][:cl.n_extra[e] * cl.extra_elem[e]].copy()
        if counts is not None:
            out["count"] = counts[:cl.n_counts].view(np.uint8).copy()
        return out


def cloud(a) -> np.ndarray:
    """float32 [N,3] → bytes-field value."""
    return np.ascontiguousarray(a, dtype=np.float32).reshape(-1).view(np.uint8).copy()


def points(v: np.ndarray) -> np.ndarray:
    """bytes-field value → float32 [N,3]."""
    return np.ascontiguousarray(v).view(np.float32).reshape(-1, 3)
