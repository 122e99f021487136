"""Classification entry points: the drop-in for the reference's classify.py.

:class:`Classifier` keeps the reference's surface (classify.py:21-128):
``Classifier(T)``, ``.classify(sigma)``, ``._run_bits(bits)``,
``.plan(raw_space)``, ``.make_scratch()``, ``.degree``, ``.maxreg``,
``.diamond``, and the module function ``classify(T, sigma, validate,
classifier)``.  Construction does the reference's once-per-triangulation
host work (reflect, sign-extension tables, antipodal pairs) and hands the
flat plan to ``tcg_plan_create``; every classification then runs on the
B200 through ``tcg_classify_batch``.  :meth:`Classifier.classify_many` and
:meth:`Classifier.classify_words` are the batched forms (one launch for
many sign vectors) that the reference has no equivalent of.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .diamond import plan_arrays, reflect
from .errors import BudgetExceeded, InvariantViolation, ParseError
from .lattice import harnack_bound, num_points, validate_triangulation
from .scheme import scheme_from_key, scheme_from_parents
from .signs import SignDistribution, free_positions

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


@dataclass(frozen=True)
class ClassificationResult:
    """Same fields and equality as the reference's (pipeline.py:240-253)."""

    scheme: str
    oval_count: int
    region_count: int
    has_pseudoline: bool

    def to_dict(self) -> dict:
        return {
            "scheme": self.scheme,
            "oval_count": self.oval_count,
            "region_count": self.region_count,
            "has_pseudoline": self.has_pseudoline,
        }


LAYOUT_MAX_DEGREE = 9  # the bit-mask kernels; larger degrees use the generic kernel


class Classifier:
    """Reusable classification state for one triangulation, resident on one GPU.

    Degrees up to 9 use the bit-mask kernels (sweeps, samples, batches);
    larger degrees -- or ``engine="generic"`` -- use the any-degree kernel
    (one CTA per patchwork), for single patchworks and batches, as the
    reference supports (sweeps are capped at d <= 9 there too).
    """

    def __init__(self, T, device: int | None = None, engine: str = "auto"):
        self.triangulation = T
        d = int(T.degree)
        self.degree = d
        D = reflect(T)
        self.diamond = D
        self.maxreg = harnack_bound(d) + 2
        self.arrays = plan_arrays(D)
        npts = num_points(d)
        rep_pos = np.full(npts, -1, dtype=np.int64)
        for pos, k in enumerate(free_positions(d)):
            rep_pos[k] = pos
        self._rep_bitpos = rep_pos
        self._raw_bitpos = np.arange(npts, dtype=np.int64)
        if engine not in ("auto", "generic", "mask"):
            raise ParseError(f"unknown engine {engine!r}")
        self.generic = engine == "generic" or (engine == "auto" and d > LAYOUT_MAX_DEGREE)
        if self.generic:
            self.native = None
            self.large = _lib.NativeLarge(self.arrays, device)
            self.device = device if device is not None else 0
        else:
            self.large = None
            self.native = _lib.NativePlan(self.arrays, device)
            self.device = self.native.info["device"]

    def device_plans(self, devices) -> list:
        """One distinct native plan per entry of ``devices`` (a device may be
        listed more than once: each entry gets its own plan, stream and
        aggregate).  Plans are created once and kept on the classifier, so
        repeated multi-device sweeps do not rebuild their device buffers."""
        if self.generic:
            raise ParseError("multi-device sweeps need the mask engine (d <= 9)")
        cache = self.__dict__.setdefault("_device_plans", {})
        seen: dict[int, int] = {}
        out = []
        for dev in devices:
            dev = int(dev)
            k = seen.get(dev, 0)
            seen[dev] = k + 1
            if dev == self.device and k == 0:
                out.append(self.native)
                continue
            if (dev, k) not in cache:
                cache[(dev, k)] = _lib.NativePlan(self.arrays, dev)
            out.append(cache[(dev, k)])
        return out

    # reference-shaped accessors -------------------------------------------
    def plan(self, raw_space: bool = False):
        """The reference's plan tuple (classify.py:53-55), for inspection."""
        a = self.arrays
        bitpos = self._raw_bitpos if raw_space else self._rep_bitpos
        return (a.degree, a.nv, a.npts, a.edge_u, a.edge_v, a.src, a.par, a.used,
                a.ap_u, a.ap_v, a.maxreg, bitpos)

    def make_scratch(self):
        """The device owns all scratch; nothing to allocate on the host."""
        return ()

    # classification ---------------------------------------------------------
    def _result(self, key, ovals, nreg, status, where: str = "") -> ClassificationResult:
        if status != 0:
            raise InvariantViolation(STATUS_MESSAGES.get(int(status), f"status {status}") + where)
        return ClassificationResult(
            scheme=scheme_from_key(int(key), self.degree % 2 == 1),
            oval_count=int(ovals),
            region_count=int(nreg),
            has_pseudoline=self.degree % 2 == 1,
        )

    def _generic_rows(self, bit_lists) -> list[ClassificationResult]:
        words = (num_points(self.degree) + 63) // 64
        rows = np.zeros((len(bit_lists), words), np.uint64)
        for t, bits in enumerate(bit_lists):
            b = np.asarray(bits, dtype=np.uint64)
            for w in range(words):
                chunk = b[64 * w: 64 * w + 64]
                rows[t, w] = np.bitwise_or.reduce(chunk << np.arange(len(chunk), dtype=np.uint64))
        st, nr, par = self.large.classify_rows(rows)
        out = []
        odd = self.degree % 2 == 1
        for t in range(len(bit_lists)):
            if st[t] != 0:
                raise InvariantViolation(STATUS_MESSAGES.get(int(st[t]), f"status {st[t]}")
                                         + (f" (at batch position {t})" if len(bit_lists) > 1
                                            else ""))
            n = int(nr[t])
            out.append(ClassificationResult(scheme_from_parents(par[t], n, odd), n - 1, n, odd))
        return out

    def _run_bits(self, bits) -> ClassificationResult:
        if self.generic:
            return self._generic_rows([bits])[0]
        b = np.asarray(bits, dtype=np.uint64)
        word = int(np.bitwise_or.reduce(b << np.arange(len(b), dtype=np.uint64))) if len(b) else 0
        key, ov, nr, st = self.native.classify_words(np.array([word], np.uint64))
        return self._result(key[0], ov[0], nr[0], st[0])

    def _sigma(self, s):
        if isinstance(s, str):
            s = SignDistribution.from_bitstring(self.degree, s)
        if s.degree != self.degree:
            raise ParseError(f"sign degree {s.degree} != triangulation degree {self.degree}")
        return s

    def classify(self, sigma) -> ClassificationResult:
        sigma = self._sigma(sigma)
        if self.generic:
            return self._generic_rows([sigma.bits])[0]
        word = 0
        for k, b in enumerate(sigma.bits):
            word |= int(b) << k
        key, ov, nr, st = self.native.classify_words(np.array([word], np.uint64))
        return self._result(key[0], ov[0], nr[0], st[0])

    def classify_words(self, words):
        """Batched raw form: uint64 sign words -> (keys, ovals, nreg, status) arrays (d <= 9)."""
        if self.generic:
            raise BudgetExceeded("uint64 sign words need d <= 9; use classify_many")
        return self.native.classify_words(words)

    def classify_many(self, sigmas) -> list[ClassificationResult]:
        sig = [self._sigma(s) for s in sigmas]
        if self.generic:
            return self._generic_rows([s.bits for s in sig]) if sig else []
        words = []
        for s in sig:
            w = 0
            for k, b in enumerate(s.bits):
                w |= int(b) << k
            words.append(w)
        key, ov, nr, st = self.native.classify_words(np.array(words, np.uint64))
        return [self._result(key[i], ov[i], nr[i], st[i], f" (at batch position {i})")
                for i in range(len(words))]


def classify(T, sigma, validate: bool = True, classifier: Classifier | None = None):
    """Classify one patchwork (reference classify.py:118-128)."""
    if validate and classifier is None:
        T = validate_triangulation(T.degree, T.edges)
    c = classifier or Classifier(T)
    return c.classify(sigma)


class MultiClassifier:
    """Many triangulations of one degree resident on one GPU (config C4).

    The reference has no multi-triangulation API; its
    equivalent is one ``Classifier(T).classify(sigma)`` per pair.  Here all
    triangulations are uploaded once and a batch of (triangulation index,
    sign vector) pairs is classified in one launch, one topology per CTA.
    """

    def __init__(self, triangulations, device: int | None = None):
        self.triangulations = list(triangulations)
        if not self.triangulations:
            raise ParseError("need at least one triangulation")
        degs = {int(T.degree) for T in self.triangulations}
        if len(degs) != 1:
            raise ParseError(f"all triangulations must share one degree, got {sorted(degs)}")
        self.degree = degs.pop()
        self.native = _lib.NativeMulti([plan_arrays(reflect(T)) for T in self.triangulations],
                                       device)

    def classify_words(self, tri, words):
        return self.native.classify_words(tri, words)

    def classify_pairs(self, pairs) -> list[ClassificationResult]:
        tri, words = [], []
        for t, s in pairs:
            if isinstance(s, str):
                s = SignDistribution.from_bitstring(self.degree, s)
            w = 0
            for k, b in enumerate(s.bits):
                w |= int(b) << k
            tri.append(int(t))
            words.append(w)
        key, ov, nr, st = self.native.classify_words(np.array(tri, np.int32),
                                                     np.array(words, np.uint64))
        odd = self.degree % 2 == 1
        out = []
        for i in range(len(words)):
            if st[i] != 0:
                raise InvariantViolation(STATUS_MESSAGES.get(int(st[i]), f"status {st[i]}")
                                         + f" (at pair {i})")
            out.append(ClassificationResult(scheme_from_key(int(key[i]), odd), int(ov[i]),
                                            int(nr[i]), odd))
        return out
