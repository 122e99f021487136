"""ctypes front-end of the CPU oracle (liboracle.so, built from tcg_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Importable
only from tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``).  See tcg_oracle.c for the reference lines each C
function restates.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

STATUS_MESSAGES = {
    1: "region count exceeds the degree bound",
    2: "even degree expects exactly one odd-cycle region, found none",
    3: "even degree expects exactly one odd-cycle region, found several",
    4: "odd degree but no pseudoline region found",
    5: "conflicting pseudoline regions",
    6: "even degree with a nonseparating curve component",
    7: "region graph is not a tree",
    8: "region graph is disconnected",
    9: "internal: canonical-string arena overflow",
    10: "internal: scheme table full",
    11: "internal: 64-bit scheme hash collision",
}


class _Plan(C.Structure):
    _fields_ = [
        ("d", C.c_int32), ("nv", C.c_int32), ("npts", C.c_int32), ("ne", C.c_int32),
        ("edge_u", C.c_void_p), ("edge_v", C.c_void_p), ("src", C.c_void_p),
        ("par", C.c_void_p), ("used", C.c_void_p),
        ("nap", C.c_int32), ("ap_u", C.c_void_p), ("ap_v", C.c_void_p),
        ("maxreg", C.c_int32),
    ]


class _Result(C.Structure):
    _fields_ = [
        ("hist", C.c_int64 * 64), ("total", C.c_int64),
        ("n", C.c_int32), ("cap", C.c_int32),
        ("count", C.c_void_p), ("witness", C.c_void_p),
        ("str_off", C.c_void_p), ("str_len", C.c_void_p),
        ("arena", C.c_void_p), ("arena_cap", C.c_int64), ("arena_used", C.c_int64),
        ("status", C.c_int32), ("bad", C.c_int64),
    ]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_sweep.argtypes = [C.POINTER(_Plan), C.c_int, C.c_int64, C.c_int64, C.c_int,
                                C.c_int64, C.POINTER(_Result)]
        L.orc_sample.argtypes = [C.POINTER(_Plan), C.c_uint64, C.c_int64, C.c_int64, C.c_int,
                                 C.c_int, C.c_int64, C.POINTER(_Result)]
        L.orc_classify_words.argtypes = [C.POINTER(_Plan), C.c_void_p, C.c_int64, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_int32]
        L.orc_classify_rows.argtypes = [C.POINTER(_Plan), C.c_void_p, C.c_int32, C.c_int64,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int32]
        L.orc_splitmix64.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_splitmix64.restype = C.c_uint64
        _lib = L
    return _lib


class OraclePlan:
    """Holds the plan arrays alive and the C struct pointing at them."""

    def __init__(self, degree, nv, npts, edge_u, edge_v, src, par, used, ap_u, ap_v, maxreg):
        self.degree = int(degree)
        self.npts = int(npts)
        self._arrs = [
            np.ascontiguousarray(edge_u, dtype=np.int32),
            np.ascontiguousarray(edge_v, dtype=np.int32),
            np.ascontiguousarray(src, dtype=np.int32),
            np.ascontiguousarray(par, dtype=np.uint8),
            np.ascontiguousarray(used, dtype=np.uint8),
            np.ascontiguousarray(ap_u, dtype=np.int32),
            np.ascontiguousarray(ap_v, dtype=np.int32),
        ]
        eu, ev, s, p, u, au, av = self._arrs
        self.c = _Plan(self.degree, int(nv), self.npts, len(eu), eu.ctypes.data, ev.ctypes.data,
                       s.ctypes.data, p.ctypes.data, u.ctypes.data, len(au), au.ctypes.data,
                       av.ctypes.data, int(maxreg))

    @classmethod
    def from_arrays(cls, P):
        """From a PlanArrays-like object (or the golden fixture dict)."""
        if isinstance(P, dict):
            return cls(P["degree"], P["nv"], P["npts"], P["edge_u"], P["edge_v"], P["src"],
                       P["par"], P["used"], P["ap_u"], P["ap_v"], P["maxreg"])
        return cls(P.degree, P.nv, P.npts, P.edge_u, P.edge_v, P.src, P.par, P.used,
                   P.ap_u, P.ap_v, P.maxreg)


def classify_words(plan: OraclePlan, words):
    """[(status, scheme|None, ovals, nreg)] for sign words (bit k = point k)."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    n = len(w)
    st = np.zeros(n, np.int32)
    ov = np.zeros(n, np.int32)
    nr = np.zeros(n, np.int32)
    sl = np.zeros(n, np.int32)
    width = 512
    buf = np.zeros(n * width, np.uint8)
    lib().orc_classify_words(C.byref(plan.c), w.ctypes.data, n, st.ctypes.data, ov.ctypes.data,
                             nr.ctypes.data, sl.ctypes.data, buf.ctypes.data, width)
    out = []
    for t in range(n):
        s = bytes(buf[t * width: t * width + sl[t]]).decode() if st[t] == 0 else None
        out.append((int(st[t]), s, int(ov[t]), int(nr[t])))
    return out


def classify_bitstrings(plan: OraclePlan, bitstrings):
    """Any degree: [(status, scheme|None, ovals, nreg)] for '0'/'1' strings."""
    words = (plan.npts + 63) // 64
    n = len(bitstrings)
    rows = np.zeros((n, words), np.uint64)
    for t, s in enumerate(bitstrings):
        for k, ch in enumerate(s):
            if ch == "1":
                rows[t, k >> 6] |= np.uint64(1) << np.uint64(k & 63)
    st = np.zeros(n, np.int32)
    ov = np.zeros(n, np.int32)
    nr = np.zeros(n, np.int32)
    sl = np.zeros(n, np.int32)
    width = 4096
    buf = np.zeros(n * width, np.uint8)
    lib().orc_classify_rows(C.byref(plan.c), rows.ctypes.data, words, n, st.ctypes.data,
                            ov.ctypes.data, nr.ctypes.data, sl.ctypes.data, buf.ctypes.data, width)
    return [(int(st[t]), bytes(buf[t * width: t * width + sl[t]]).decode() if st[t] == 0 else None,
             int(ov[t]), int(nr[t])) for t in range(n)]


def _run(fn, plan, *args, cap=1 << 16):
    count = np.zeros(cap, np.int64)
    wit = np.zeros(cap, np.int64)
    off = np.zeros(cap, np.int64)
    ln = np.zeros(cap, np.int32)
    arena = np.zeros(cap * 64, np.uint8)
    R = _Result()
    R.cap = cap
    R.count, R.witness, R.str_off, R.str_len = (count.ctypes.data, wit.ctypes.data,
                                                off.ctypes.data, ln.ctypes.data)
    R.arena, R.arena_cap = arena.ctypes.data, len(arena)
    fn(C.byref(plan.c), *args, C.byref(R))
    schemes = {}
    for q in range(R.n):
        s = bytes(arena[off[q]: off[q] + ln[q]]).decode()
        schemes[s] = (int(count[q]), int(wit[q]))
    return {
        "hist": [int(x) for x in R.hist],
        "schemes": schemes,
        "total": int(R.total),
        "status": int(R.status),
        "bad": int(R.bad),
    }


def sweep(plan: OraclePlan, raw: bool, start: int, end: int, threads: int = 1,
          chunk: int = 1 << 16):
    return _run(lib().orc_sweep, plan, int(raw), int(start), int(end), int(threads), int(chunk))


def sample(plan: OraclePlan, seed: int, k0: int, k1: int, nbits: int, threads: int = 1,
           chunk: int = 1 << 16):
    return _run(lib().orc_sample, plan, int(seed) & (2**64 - 1), int(k0), int(k1), int(nbits),
                int(threads), int(chunk))


def splitmix64(seed: int, k: int) -> int:
    return int(lib().orc_splitmix64(int(seed) & (2**64 - 1), int(k)))
