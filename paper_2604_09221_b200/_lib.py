"""ctypes binding of libtcg.so (the sm_100a classifier, csrc/tcg.cu).

This is the only door to the device: there is no CPU fallback.  If the
library is missing, was built for another architecture, or no CUDA device
is present, every entry point raises :class:`DeviceUnavailable` /
:class:`DeviceError` loudly.  The library is built in-tree by
``__graft_entry__.build()`` (nvcc -gencode arch=compute_100a,code=sm_100a).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import BudgetExceeded, DeviceError, DeviceUnavailable, IndexOutOfRange

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TCG_LIBRARY", os.path.join(HERE, "libtcg.so"))

TCG_E_ARG, TCG_E_CUDA, TCG_E_UNSUPPORTED, TCG_E_RANGE = -1, -2, -3, -4
AGG_CAP = 1 << 16


class TcgDesc(C.Structure):
    _fields_ = [
        ("degree", C.c_int32), ("nv", C.c_int32), ("npts", C.c_int32), ("ne", C.c_int32),
        ("edge_u", C.c_void_p), ("edge_v", C.c_void_p), ("src", C.c_void_p),
        ("par", C.c_void_p), ("used", C.c_void_p),
        ("nap", C.c_int32), ("ap_u", C.c_void_p), ("ap_v", C.c_void_p),
        ("maxreg", C.c_int32),
    ]


class TcgAgg(C.Structure):
    _fields_ = [
        ("hist", C.c_int64 * 64), ("total", C.c_int64),
        ("n", C.c_int32), ("cap", C.c_int32),
        ("key", C.c_void_p), ("count", C.c_void_p), ("witness", C.c_void_p),
    ]


_lib = None
_lock = threading.Lock()


def load():
    """Load libtcg.so once; raise DeviceUnavailable if it cannot be used."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailable(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.tcg_plan_create.argtypes = [C.POINTER(TcgDesc), C.c_int, C.POINTER(P)]
        L.tcg_plan_destroy.argtypes = [P]
        L.tcg_plan_set_stream.argtypes = [P, C.c_void_p]
        L.tcg_plan_info.argtypes = [P, C.c_void_p, C.c_int]
        L.tcg_plan_set_timing.argtypes = [P, C.c_int]
        L.tcg_kernel_times.argtypes = [P, C.c_void_p, C.c_void_p]
        L.tcg_plan_set_dedup.argtypes = [P, C.c_int]
        L.tcg_tile_stats.argtypes = [P, C.c_void_p]
        L.tcg_plan_set_level2.argtypes = [P, C.c_int]
        L.tcg_level2_stats.argtypes = [P, C.c_void_p]
        L.tcg_plan_set_split.argtypes = [P, C.c_int]
        L.tcg_split_stats.argtypes = [P, C.c_void_p]
        L.tcg_split_design.argtypes = [C.POINTER(TcgDesc), C.c_void_p]
        L.tcg_classify_batch.argtypes = [P, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p]
        L.tcg_classify_batch_device.argtypes = L.tcg_classify_batch.argtypes
        L.tcg_sweep.argtypes = [P, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(TcgAgg),
                                C.POINTER(C.c_int64)]
        L.tcg_sample.argtypes = [P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                 C.POINTER(TcgAgg), C.POINTER(C.c_int64)]
        L.tcg_agg_reset.argtypes = [P]
        L.tcg_sweep_async.argtypes = [P, C.c_int, C.c_uint64, C.c_uint64]
        L.tcg_sample_async.argtypes = [P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        L.tcg_agg_fetch.argtypes = [P, C.POINTER(TcgAgg), C.POINTER(C.c_int64)]
        L.tcg_sweep_multi.argtypes = [C.POINTER(P), C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                      C.POINTER(TcgAgg), C.POINTER(C.c_int64)]
        L.tcg_sample_multi.argtypes = [C.POINTER(P), C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_int, C.POINTER(TcgAgg), C.POINTER(C.c_int64)]
        L.tcg_last_error.restype = C.c_char_p
        L.tcg_version.restype = C.c_char_p
        L.tcg_device_count.restype = C.c_int
        L.tcg_launch_count.argtypes = [P]
        L.tcg_launch_count.restype = C.c_int64
        L.tcg_multi_create.argtypes = [C.POINTER(TcgDesc), C.c_int32, C.c_int, C.POINTER(P)]
        L.tcg_multi_destroy.argtypes = [P]
        L.tcg_multi_classify.argtypes = [P, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.tcg_multi_last_ms.argtypes = [P]
        L.tcg_multi_last_ms.restype = C.c_double
        L.tcg_large_create.argtypes = [C.POINTER(TcgDesc), C.c_int, C.POINTER(P)]
        L.tcg_large_destroy.argtypes = [P]
        L.tcg_large_classify.argtypes = [P, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        _lib = L
        return L


EXPORTS = (
    "tcg_plan_create", "tcg_plan_destroy", "tcg_plan_set_stream", "tcg_plan_info",
    "tcg_plan_set_timing", "tcg_kernel_times", "tcg_plan_set_dedup", "tcg_tile_stats",
    "tcg_plan_set_level2", "tcg_level2_stats", "tcg_plan_set_split", "tcg_split_stats", "tcg_split_design",
    "tcg_classify_batch", "tcg_classify_batch_device", "tcg_sweep", "tcg_sample",
    "tcg_agg_reset", "tcg_sweep_async", "tcg_sample_async", "tcg_agg_fetch",
    "tcg_sweep_multi", "tcg_sample_multi", "tcg_last_error", "tcg_device_count",
    "tcg_launch_count", "tcg_version", "tcg_multi_create", "tcg_multi_destroy",
    "tcg_multi_classify", "tcg_multi_last_ms", "tcg_large_create", "tcg_large_destroy",
    "tcg_large_classify",
)


# tcg.h TCG_KT_* order (tcg_kernel_times)
KERNEL_KINDS = ("tile_build", "tile_classify", "enumerate", "batch", "tile_dedup",
                "l2_build", "l2_dedup", "l2_classify", "super_build", "l15_build", "l15_dedup",
                "split_build", "sample_split", "sample_list")


def last_error() -> str:
    return load().tcg_last_error().decode(errors="replace")


def device_count() -> int:
    return int(load().tcg_device_count())


def _check(rc: int, what: str):
    if rc == 0:
        return
    msg = f"{what}: {last_error()}"
    if rc == TCG_E_UNSUPPORTED:
        raise BudgetExceeded(msg)
    if rc == TCG_E_RANGE:
        raise IndexOutOfRange(msg)
    if rc == TCG_E_CUDA:
        raise DeviceError(msg)
    raise DeviceError(f"{msg} (code {rc})")


class AggBuffers:
    """Host-side tcg_agg with caller-owned arrays."""

    def __init__(self, cap: int = AGG_CAP):
        self.key = np.zeros(cap, np.uint64)
        self.count = np.zeros(cap, np.int64)
        self.witness = np.zeros(cap, np.int64)
        self.c = TcgAgg()
        self.c.cap = cap
        self.c.key = self.key.ctypes.data
        self.c.count = self.count.ctypes.data
        self.c.witness = self.witness.ctypes.data

    def result(self):
        n = self.c.n
        return (
            [int(x) for x in self.c.hist],
            int(self.c.total),
            self.key[:n].copy(),
            self.count[:n].copy(),
            self.witness[:n].copy(),
        )


def _desc(arrays, keep):
    arrs = [
        np.ascontiguousarray(arrays.edge_u, np.int32),
        np.ascontiguousarray(arrays.edge_v, np.int32),
        np.ascontiguousarray(arrays.src, np.int32),
        np.ascontiguousarray(arrays.par, np.uint8),
        np.ascontiguousarray(arrays.used, np.uint8),
        np.ascontiguousarray(arrays.ap_u, np.int32),
        np.ascontiguousarray(arrays.ap_v, np.int32),
    ]
    keep.extend(arrs)
    eu, ev, src, par, used, apu, apv = arrs
    return TcgDesc(arrays.degree, arrays.nv, arrays.npts, len(eu), eu.ctypes.data,
                   ev.ctypes.data, src.ctypes.data, par.ctypes.data, used.ctypes.data,
                   len(apu), apu.ctypes.data, apv.ctypes.data, arrays.maxreg)


def split_design(arrays):
    """The split sampler's separator for a plan, computed on the host (no GPU):
    None if it does not apply, else a dict (tcg.h tcg_split_design)."""
    L = load()
    keep = []
    d = _desc(arrays, keep)
    out = np.zeros(9, np.int64)
    _check(L.tcg_split_design(C.byref(d), out.ctypes.data), "tcg_split_design")
    if not out[0]:
        return None
    u = [int(x) & ((1 << 64) - 1) for x in out]
    return {"separator_vertices": u[1], "bits_a": u[2], "bits_b": u[3], "F": u[4], "A": u[5],
            "B": u[6], "mean_nodes": u[7] / 1000.0, "table_bytes": u[8]}


class NativeMulti:
    """Owns one tcg_multi (many triangulations of one degree on one device)."""

    def __init__(self, arrays_list, device: int | None = None):
        L = load()
        if L.tcg_device_count() < 1:
            raise DeviceUnavailable("no CUDA device visible; the classifier has no CPU fallback")
        self._keep = []
        descs = (TcgDesc * len(arrays_list))(*[_desc(a, self._keep) for a in arrays_list])
        h = C.c_void_p()
        _check(L.tcg_multi_create(descs, len(arrays_list), -1 if device is None else int(device),
                                  C.byref(h)), "tcg_multi_create")
        self.h = h
        self._L = L
        self.ntri = len(arrays_list)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                self._L.tcg_multi_destroy(h)
            except Exception:
                pass
            self.h = None

    def classify_words(self, tri, words):
        t = np.ascontiguousarray(tri, dtype=np.int32)
        w = np.ascontiguousarray(words, dtype=np.uint64)
        n = len(w)
        if len(t) != n:
            raise ValueError("tri and words must have the same length")
        key = np.empty(n, np.uint64)
        ov = np.empty(n, np.uint8)
        nr = np.empty(n, np.uint8)
        st = np.empty(n, np.int32)
        if n:
            _check(self._L.tcg_multi_classify(self.h, t.ctypes.data, w.ctypes.data, n,
                                              key.ctypes.data, ov.ctypes.data, nr.ctypes.data,
                                              st.ctypes.data), "tcg_multi_classify")
        return key, ov, nr, st

    def last_ms(self) -> float:
        return float(self._L.tcg_multi_last_ms(self.h))


class NativeLarge:
    """Owns one tcg_large (any degree; one CTA per patchwork)."""

    def __init__(self, arrays, device: int | None = None):
        L = load()
        if L.tcg_device_count() < 1:
            raise DeviceUnavailable("no CUDA device visible; the classifier has no CPU fallback")
        self._keep = []
        desc = _desc(arrays, self._keep)
        h = C.c_void_p()
        _check(L.tcg_large_create(C.byref(desc), -1 if device is None else int(device),
                                  C.byref(h)), "tcg_large_create")
        self.h = h
        self._L = L
        self.maxreg = int(arrays.maxreg)
        self.words = (int(arrays.npts) + 63) // 64

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                self._L.tcg_large_destroy(h)
            except Exception:
                pass
            self.h = None

    def classify_rows(self, rows):
        """rows: uint64 [n, words] sign bit rows -> (status, nreg, parent [n, maxreg])."""
        r = np.ascontiguousarray(rows, dtype=np.uint64).reshape(-1, self.words)
        n = r.shape[0]
        st = np.zeros(n, np.int32)
        nr = np.zeros(n, np.int32)
        par = np.full((n, self.maxreg), -1, np.int32)
        if n:
            _check(self._L.tcg_large_classify(self.h, r.ctypes.data, n, st.ctypes.data,
                                              nr.ctypes.data, par.ctypes.data),
                   "tcg_large_classify")
        return st, nr, par


class NativePlan:
    """Owns one tcg_plan (one triangulation on one device)."""

    def __init__(self, arrays, device: int | None = None):
        L = load()
        if device is None:
            device = -1
        if L.tcg_device_count() < 1:
            raise DeviceUnavailable("no CUDA device visible; the classifier has no CPU fallback")
        self.arrays = arrays
        self._keep = [
            np.ascontiguousarray(arrays.edge_u, np.int32),
            np.ascontiguousarray(arrays.edge_v, np.int32),
            np.ascontiguousarray(arrays.src, np.int32),
            np.ascontiguousarray(arrays.par, np.uint8),
            np.ascontiguousarray(arrays.used, np.uint8),
            np.ascontiguousarray(arrays.ap_u, np.int32),
            np.ascontiguousarray(arrays.ap_v, np.int32),
        ]
        eu, ev, src, par, used, apu, apv = self._keep
        desc = TcgDesc(arrays.degree, arrays.nv, arrays.npts, len(eu), eu.ctypes.data,
                       ev.ctypes.data, src.ctypes.data, par.ctypes.data, used.ctypes.data,
                       len(apu), apu.ctypes.data, apv.ctypes.data, arrays.maxreg)
        h = C.c_void_p()
        _check(L.tcg_plan_create(C.byref(desc), int(device), C.byref(h)), "tcg_plan_create")
        self.h = h
        self._L = L
        info = np.zeros(10, np.int32)
        L.tcg_plan_info(self.h, info.ctypes.data, 10)
        self.info = {
            "degree": int(info[0]), "words": int(info[1]), "used": int(info[2]),
            "device": int(info[3]), "sms": int(info[4]), "ctas": int(info[5]),
            "threads": int(info[6]), "maxreg": int(info[7]), "tile_bits_raw": int(info[8]),
            "tile_bits_rep": int(info[9]),
        }

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                self._L.tcg_plan_destroy(h)
            except Exception:
                pass
            self.h = None

    def set_stream(self, stream_handle: int | None):
        _check(self._L.tcg_plan_set_stream(self.h, C.c_void_p(stream_handle or 0)),
               "tcg_plan_set_stream")

    def launches(self) -> int:
        return int(self._L.tcg_launch_count(self.h))

    def set_timing(self, enable: bool):
        _check(self._L.tcg_plan_set_timing(self.h, int(bool(enable))), "tcg_plan_set_timing")

    def kernel_times(self):
        """{kind: (ms, launches)} since the last call; kinds as in tcg.h."""
        names = KERNEL_KINDS
        ms = np.zeros(len(names), np.float64)
        n = np.zeros(len(names), np.int64)
        _check(self._L.tcg_kernel_times(self.h, ms.ctypes.data, n.ctypes.data), "tcg_kernel_times")
        return {names[i]: (float(ms[i]), int(n[i])) for i in range(len(names))}

    def set_dedup(self, enable: bool | None):
        """Tile deduplication on / off / None = default (see tcg.h)."""
        flag = -1 if enable is None else int(bool(enable))
        _check(self._L.tcg_plan_set_dedup(self.h, flag), "tcg_plan_set_dedup")

    def set_level2(self, enable: bool | None):
        """Level-2 contraction on / off / None = default (see tcg.h)."""
        flag = -1 if enable is None else int(bool(enable))
        _check(self._L.tcg_plan_set_level2(self.h, flag), "tcg_plan_set_level2")

    def level2_stats(self):
        """(level-2 records built, level-2 records classified, tiles left to the
        level-1 classifier while level 2 ran) since the last call."""
        out = np.zeros(3, np.int64)
        _check(self._L.tcg_level2_stats(self.h, out.ctypes.data), "tcg_level2_stats")
        return int(out[0]), int(out[1]), int(out[2])

    def set_split(self, enable: bool | None):
        """Separator-split sampling on / off / None = default (see tcg.h)."""
        flag = -1 if enable is None else int(bool(enable))
        _check(self._L.tcg_plan_set_split(self.h, flag), "tcg_plan_set_split")

    def split_stats(self):
        """(state, draws through the split kernel, of those left to the flat
        kernel, separator vertices, table bytes); counts since the last call."""
        out = np.zeros(5, np.int64)
        _check(self._L.tcg_split_stats(self.h, out.ctypes.data), "tcg_split_stats")
        return tuple(int(x) for x in out)

    def tile_stats(self):
        """(tiles contracted, tiles classified) since the last call."""
        out = np.zeros(2, np.int64)
        _check(self._L.tcg_tile_stats(self.h, out.ctypes.data), "tcg_tile_stats")
        return int(out[0]), int(out[1])

    def classify_words(self, words):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        n = len(w)
        key = np.empty(n, np.uint64)
        ov = np.empty(n, np.uint8)
        nr = np.empty(n, np.uint8)
        st = np.empty(n, np.int32)
        if n:
            _check(self._L.tcg_classify_batch(self.h, w.ctypes.data, n, key.ctypes.data,
                                              ov.ctypes.data, nr.ctypes.data, st.ctypes.data),
                   "tcg_classify_batch")
        return key, ov, nr, st

    def classify_words_device(self, d_sig: int, n: int, d_key: int, d_ov: int, d_nr: int,
                              d_st: int):
        _check(self._L.tcg_classify_batch_device(self.h, d_sig, n, d_key, d_ov, d_nr, d_st),
               "tcg_classify_batch_device")

    def sweep(self, raw: bool, start: int, end: int, agg: AggBuffers | None = None):
        agg = agg or AggBuffers()
        bad = C.c_int64(-1)
        rc = self._L.tcg_sweep(self.h, int(bool(raw)), int(start), int(end), C.byref(agg.c),
                               C.byref(bad))
        if rc < 0:
            _check(rc, "tcg_sweep")
        return rc, int(bad.value), agg

    def sample(self, seed: int, k0: int, k1: int, nbits: int, agg: AggBuffers | None = None):
        agg = agg or AggBuffers()
        bad = C.c_int64(-1)
        rc = self._L.tcg_sample(self.h, int(seed) & (2**64 - 1), int(k0), int(k1), int(nbits),
                                C.byref(agg.c), C.byref(bad))
        if rc < 0:
            _check(rc, "tcg_sample")
        return rc, int(bad.value), agg

    # split phase (bench, distributed shards)
    def agg_reset(self):
        _check(self._L.tcg_agg_reset(self.h), "tcg_agg_reset")

    def sweep_async(self, raw: bool, start: int, end: int):
        _check(self._L.tcg_sweep_async(self.h, int(bool(raw)), int(start), int(end)),
               "tcg_sweep_async")

    def sample_async(self, seed: int, k0: int, k1: int, nbits: int):
        _check(self._L.tcg_sample_async(self.h, int(seed) & (2**64 - 1), int(k0), int(k1),
                                        int(nbits)), "tcg_sample_async")

    def agg_fetch(self, agg: AggBuffers | None = None):
        agg = agg or AggBuffers()
        bad = C.c_int64(-1)
        rc = self._L.tcg_agg_fetch(self.h, C.byref(agg.c), C.byref(bad))
        if rc < 0:
            _check(rc, "tcg_agg_fetch")
        return rc, int(bad.value), agg


def sweep_multi(plans, raw, start, end, agg: AggBuffers | None = None):
    L = load()
    agg = agg or AggBuffers()
    arr = (C.c_void_p * len(plans))(*[p.h.value for p in plans])
    bad = C.c_int64(-1)
    rc = L.tcg_sweep_multi(arr, len(plans), int(bool(raw)), int(start), int(end), C.byref(agg.c),
                           C.byref(bad))
    if rc < 0:
        _check(rc, "tcg_sweep_multi")
    return rc, int(bad.value), agg


def sample_multi(plans, seed, k0, k1, nbits, agg: AggBuffers | None = None):
    L = load()
    agg = agg or AggBuffers()
    arr = (C.c_void_p * len(plans))(*[p.h.value for p in plans])
    bad = C.c_int64(-1)
    rc = L.tcg_sample_multi(arr, len(plans), int(seed) & (2**64 - 1), int(k0), int(k1),
                            int(nbits), C.byref(agg.c), C.byref(bad))
    if rc < 0:
        _check(rc, "tcg_sample_multi")
    return rc, int(bad.value), agg
