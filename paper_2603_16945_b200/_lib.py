"""ctypes binding of libpcpipe_b200.so (include/pcpipe_b200.h).

The Python side mirrors the reference's pipeline interface
(proj/core/include/pcpipe/pipeline.hpp:157-186): a ``Pipeline`` built from
the graph JSON, ``next_batch()`` returning batches in dataset order, ``None``
at the end, and worker failures raised as ``PcError(kWorkerPanic)``.  All
compute happens in the CUDA library; if it is missing or no sm_100 device is
present, constructing a Pipeline raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpcpipe_b200.so")

ERRC = ["OK", "DuplicateField", "EmptySchema", "BadShape", "BadAlignment", "ColumnOutOfRange",
        "ChecksumMismatch", "CorruptPage", "SchemaMismatch", "IoFailure", "EmptyDataset",
        "BadMagic", "UnsupportedVersion", "CorruptHeader", "RangeOutOfBounds", "SchemaConflict",
        "OutOfRange", "NotPadded", "MalformedHeader", "TruncatedPayload", "UnsupportedProperty",
        "NoInputFiles", "ParseFailure", "Shutdown", "MissingField", "EmptyCloud", "UnknownOp",
        "OutOfBounds", "WorkerPanic", "ShapeMismatch"]
K = {name: i for i, name in enumerate(ERRC)}  # status = Errc + 1

_DTYPE_OF_KIND = {0: np.uint8, 1: np.int32, 2: np.int64, 3: np.float32, 4: np.float64}
_KIND_OF_DTYPE = {np.dtype(np.uint8): 0, np.dtype(np.int32): 1, np.dtype(np.int64): 2,
                  np.dtype(np.float32): 3, np.dtype(np.float64): 4}


class PcError(RuntimeError):
    """Mirror of pcpipe::PcError: ``code`` is the C-ABI status (Errc + 1)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code

    @property
    def errc(self) -> str:
        return ERRC[self.code] if 0 <= self.code < len(ERRC) else "Unknown"


class _Field(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("kind", C.c_int32), ("d_ptr", C.c_void_p),
                ("nbytes", C.c_uint64), ("h_offsets", C.POINTER(C.c_uint64)),
                ("uniform", C.c_int32), ("h_ptr", C.c_void_p)]


class _Batch(C.Structure):
    _fields_ = [("epoch", C.c_uint64), ("batch_index", C.c_uint64), ("n_samples", C.c_uint32),
                ("n_fields", C.c_uint32), ("fields", _Field * 16)]


_lib = None

# pcp_page_source_fn / pcp_wave_done_fn (include/pcpipe_b200.h)
PAGE_SOURCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint8))
WAVE_DONE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64)


def lib():
    """Load the CUDA library (built by ``make -C paper_2603_16945_b200``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PcError(K["IoFailure"], f"{LIB_PATH} is not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.pcp_last_error.restype = C.c_char_p
        L.pcp_errc_name.restype = C.c_char_p
        L.pcp_mix_seed.restype = C.c_uint64
        L.pcp_mix_seed.argtypes = [C.c_uint64] * 4
        L.pcp_map_kind_from_name.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.pcp_write_dataset.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t,
                                        C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
        L.pcp_write_dataset_device.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t,
                                               C.c_uint32, C.c_uint32, C.c_uint32, C.c_int]
        L.pcp_pipeline_open.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_uint64), C.c_uint64,
                                        C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]
        L.pcp_pipeline_open_source.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.POINTER(C.c_uint64),
                                               C.c_uint64, C.c_int, C.c_char_p, PAGE_SOURCE_FN, WAVE_DONE_FN,
                                               C.c_void_p, C.POINTER(C.c_void_p)]
        L.pcp_pipeline_next_batch.argtypes = [C.c_void_p, C.POINTER(_Batch), C.POINTER(C.c_int)]
        L.pcp_pipeline_stream.restype = C.c_void_p
        L.pcp_pipeline_stream.argtypes = [C.c_void_p]
        L.pcp_pipeline_stats.restype = C.c_char_p
        L.pcp_pipeline_stats.argtypes = [C.c_void_p]
        L.pcp_pipeline_close.argtypes = [C.c_void_p]
        L.pcp_pipeline_metrics.restype = C.c_char_p
        L.pcp_pipeline_metrics.argtypes = [C.c_void_p]
        L.pcp_pipeline_update_config.argtypes = [C.c_void_p, C.c_char_p]
        L.pcp_memcpy_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.pcp_memcpy_d2h_async.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.pcp_memcpy_h2d.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.pcp_device_info.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int)]
        _lib = L
    return _lib


def _check(st: int):
    if st:
        raise PcError(st, lib().pcp_last_error().decode())


def mix_seed(base: int, epoch: int, index: int, op_id: int) -> int:
    return lib().pcp_mix_seed(base, epoch, index, op_id)


def map_kind_from_name(name: str) -> int:
    k = C.c_int()
    _check(lib().pcp_map_kind_from_name(name.encode(), C.byref(k)))
    return k.value


def device_info(device: int = 0):
    sm, ma, mi = C.c_int(), C.c_int(), C.c_int()
    _check(lib().pcp_device_info(device, C.byref(sm), C.byref(ma), C.byref(mi)))
    return {"sm_count": sm.value, "cc": (ma.value, mi.value)}


def encode_samples(samples: list) -> bytes:
    out = []
    for s in samples:
        out.append(struct.pack("<I", len(s)))
        for name in sorted(s):
            v = s[name]
            nb = name.encode()
            if isinstance(v, str):
                kind, raw = 5, v.encode()
            else:
                a = np.ascontiguousarray(v)
                kind, raw = _KIND_OF_DTYPE[a.dtype], a.tobytes()
            out.append(struct.pack("<H", len(nb)) + nb + struct.pack("<BQ", kind, len(raw)) + raw)
    return b"".join(out)


def write_dataset(out_dir, stem: str, schema: dict, samples: list, slice_count: int = 1,
                  group_size: int = 256, n_threads: int = 0, device: int | None = None) -> str:
    """write_dataset (format.cpp:499-610), byte-identical to the reference;
    ``device``: encode the pages on that GPU (pcp_write_dataset_device)."""
    tlv = encode_samples(samples)
    if device is None:
        _check(lib().pcp_write_dataset(str(out_dir).encode(), stem.encode(), json.dumps(schema).encode(),
                                       tlv, len(tlv), len(samples), slice_count, group_size, n_threads))
    else:
        _check(lib().pcp_write_dataset_device(str(out_dir).encode(), stem.encode(), json.dumps(schema).encode(),
                                              tlv, len(tlv), len(samples), slice_count, group_size, device))
    return os.path.join(str(out_dir), stem + ".pcrecord")


class DeviceBatch:
    """One batch as device views.  ``fields[name] = (kind, d_ptr, nbytes,
    offsets, uniform)``; offsets are per-sample byte offsets (CSR)."""

    def __init__(self, b: _Batch, stream):
        self.epoch = b.epoch
        self.batch_index = b.batch_index
        self.n_samples = b.n_samples
        self.stream = stream
        self.fields = {}
        for i in range(b.n_fields):
            f = b.fields[i]
            offs = np.ctypeslib.as_array(f.h_offsets, shape=(b.n_samples + 1,)).copy()
            self.fields[f.name.decode()] = (f.kind, f.d_ptr, f.nbytes, offs, bool(f.uniform))

    @property
    def h2d_free_bytes(self) -> int:
        return sum(v[2] for v in self.fields.values())

    def to_host(self, into: dict | None = None) -> dict:
        """Copy every field to host numpy arrays (stacked layout)."""
        out = {}
        for name, (kind, ptr, nbytes, offs, _) in self.fields.items():
            dt = _DTYPE_OF_KIND.get(kind, np.uint8)
            if into is not None and name in into:
                buf = into[name]
            else:
                buf = np.empty(nbytes, dtype=np.uint8)
            if nbytes:
                _check(lib().pcp_memcpy_d2h(buf.ctypes.data, ptr, nbytes, self.stream))
            out[name] = (buf[:nbytes].view(dt) if kind != 5 else buf[:nbytes], offs)
        return out

    def samples(self) -> list:
        """Per-sample dicts like the reference Batch.samples (values as numpy)."""
        host = self.to_host()
        res = [dict() for _ in range(self.n_samples)]
        for name, (arr, offs) in host.items():
            kind = self.fields[name][0]
            raw = arr.view(np.uint8) if kind != 5 else arr
            for k in range(self.n_samples):
                chunk = raw[offs[k]:offs[k + 1]]
                if kind == 5:
                    res[k][name] = bytes(chunk).decode()
                else:
                    res[k][name] = chunk.view(_DTYPE_OF_KIND[kind]).copy()
        return res


class Pipeline:
    """B200 PcRecord → batch pipeline (drop-in for pcpipe::Pipeline on this
    path).  ``graph`` is the reference graph JSON (dict or str)."""

    def __init__(self, primary, graph, ids=None, device: int = 0, epochs: int = 1,
                 resident: bool = True, wave_batches: int = 0, force_serial_fy: bool = False,
                 slots: int | None = None, host_batches: bool = False, **options):
        L = lib()
        g = graph if isinstance(graph, str) else json.dumps(graph)
        o = {"epochs": epochs, "resident": resident, "wave_batches": wave_batches,
             "force_serial_fy": force_serial_fy, "host_batches": host_batches, **options}
        if slots is not None:
            o["slots"] = slots
        opts = json.dumps(o)
        h = C.c_void_p()
        if ids is None:
            p, n = None, 0
        else:
            self._ids = np.ascontiguousarray(ids, dtype=np.uint64)
            p, n = self._ids.ctypes.data_as(C.POINTER(C.c_uint64)), len(self._ids)
        _check(L.pcp_pipeline_open(str(primary).encode(), g.encode(), p, n, device, opts.encode(),
                                   C.byref(h)))
        self._h = h
        self.stream = L.pcp_pipeline_stream(h)

    @classmethod
    def from_source(cls, header: bytes, graph, read, done=None, ids=None, device: int = 0,
                    epochs: int = 1, **options):
        """Pipeline over caller-supplied pages (pcp_pipeline_open_source, the
        SourceFn analogue): ``read(slice, offset, length) -> bytes`` may block
        until the slice is present; ``done(epoch, first_index, count)`` is
        called once those walk positions' pages are on the device."""
        self = cls.__new__(cls)
        L = lib()
        g = graph if isinstance(graph, str) else json.dumps(graph)
        opts = json.dumps({"epochs": epochs, **options})

        def _read(_user, sl, off, n, dst):
            try:
                b = read(sl, off, n)
                if len(b) != n:
                    return K["IoFailure"]
                C.memmove(dst, b, n)
                return 0
            except Exception:
                return K["IoFailure"]

        self._read_cb = PAGE_SOURCE_FN(_read)
        self._done_cb = WAVE_DONE_FN(lambda _u, e, f, n: done(e, f, n)) if done else WAVE_DONE_FN()
        h = C.c_void_p()
        if ids is None:
            p, n = None, 0
        else:
            self._ids = np.ascontiguousarray(ids, dtype=np.uint64)
            p, n = self._ids.ctypes.data_as(C.POINTER(C.c_uint64)), len(self._ids)
        _check(L.pcp_pipeline_open_source(header, len(header), g.encode(), p, n, device, opts.encode(),
                                          self._read_cb, self._done_cb, None, C.byref(h)))
        self._h = h
        self.stream = L.pcp_pipeline_stream(h)
        return self

    def next_batch(self) -> DeviceBatch | None:
        b = _Batch()
        eos = C.c_int()
        _check(lib().pcp_pipeline_next_batch(self._h, C.byref(b), C.byref(eos)))
        if eos.value:
            return None
        return DeviceBatch(b, self.stream)

    def next_batch_raw(self):
        """The bare pcp_pipeline_next_batch call (what a C++ GpuPipeline makes):
        returns the library's batch struct — reused, valid until the next call —
        or None at the end.  For throughput loops that need no Python objects."""
        if not hasattr(self, "_raw"):
            self._raw, self._eos = _Batch(), C.c_int()
            self._next = lib().pcp_pipeline_next_batch
        _check(self._next(self._h, C.byref(self._raw), C.byref(self._eos)))
        return None if self._eos.value else self._raw

    def next_host_batch(self) -> dict | None:
        """host_batches pipelines: the next batch as ``{name: (array, offsets)}``
        copied out of the library's pinned wave buffer (the layout of
        ``DeviceBatch.to_host``), or None at the end."""
        b = self.next_batch_raw()
        if b is None:
            return None
        out = {}
        for i in range(b.n_fields):
            f = b.fields[i]
            if not f.h_ptr and f.nbytes:
                raise PcError(1, "pipeline was not opened with host_batches")
            kind = f.kind
            raw = np.ctypeslib.as_array(C.cast(f.h_ptr, C.POINTER(C.c_uint8)), shape=(f.nbytes,)).copy() \
                if f.nbytes else np.empty(0, np.uint8)
            offs = np.ctypeslib.as_array(f.h_offsets, shape=(b.n_samples + 1,)).copy()
            out[f.name.decode()] = (raw.view(_DTYPE_OF_KIND.get(kind, np.uint8)) if kind != 5 else raw, offs)
        return out

    def __iter__(self):
        while True:
            b = self.next_batch()
            if b is None:
                return
            yield b

    def stats(self) -> dict:
        return json.loads(lib().pcp_pipeline_stats(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            lib().pcp_pipeline_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def run_pipeline(primary, graph, ids=None, epochs: int = 1, **kw) -> list:
    """run_pipeline (pipeline.cpp:808-824): every batch as per-sample dicts."""
    out = []
    with Pipeline(primary, graph, ids=ids, epochs=epochs, **kw) as p:
        for b in p:
            out.append({"epoch": b.epoch, "batch_index": b.batch_index, "samples": b.samples()})
    return out
