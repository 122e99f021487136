"""Exhaustive sweeps and seeded sampling on the GPU (drop-in for sweep.py).

Same API, domains and report semantics as the reference (sweep.py:35-252):
the representative domain 2^(|A|-3) by default, the raw 2^|A| domain with
``raw_space=True``, indices capped at 62 bits, sampling by the counter
generator ``m_k = splitmix64(seed, k) & (2^(|A|-3) - 1)`` over
representatives, reports merged by count sum and witness minimum.

Differences: ``workers`` and ``chunk_size`` are accepted for signature
compatibility and do not change the result (the reference guarantees the
same invariance, sweep.py:1-11); the work runs on the GPU as one call to
``tcg_sweep`` / ``tcg_sample``.  ``devices=[...]`` shards the range over
several GPUs of one process (``tcg_sweep_multi``); for one process per GPU
see :mod:`.distributed`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .classify import STATUS_MESSAGES, Classifier
from .errors import BudgetExceeded, IndexOutOfRange, InvariantViolation, MergeMismatch
from .lattice import fingerprint_of, harnack_bound, num_points
from .scheme import scheme_from_key
from .signs import representative, sign_from_raw_index

DEFAULT_CHUNK = 1 << 16
_MAX_DOMAIN_BITS = 62


@dataclass(frozen=True)
class SweepRange:
    start: int
    end: int

    def __post_init__(self):
        if not (0 <= self.start <= self.end):
            raise IndexOutOfRange(f"bad sweep range [{self.start}, {self.end})")


@dataclass
class SweepReport:
    """Mergeable aggregate of one enumeration run (reference sweep.py:45-69)."""

    degree: int
    fingerprint: str
    raw_space: bool
    oval_histogram: tuple[int, ...]
    scheme_map: dict[str, tuple[int, int]]
    total_classified: int
    params: dict = field(default_factory=dict, compare=False)

    def witness_bitstring(self, scheme: str) -> str:
        m = self.scheme_map[scheme][1]
        if self.raw_space:
            return sign_from_raw_index(self.degree, m).bitstring()
        return representative(self.degree, m).bitstring()

    def distinct_schemes(self) -> int:
        return len(self.scheme_map)

    def max_ovals(self) -> int:
        return max((k for k, c in enumerate(self.oval_histogram) if c), default=0)


def empty_report(T, raw_space: bool = False) -> SweepReport:
    return SweepReport(
        degree=T.degree,
        fingerprint=fingerprint_of(T),
        raw_space=raw_space,
        oval_histogram=tuple([0] * (harnack_bound(T.degree) + 1)),
        scheme_map={},
        total_classified=0,
    )


def merge(a: SweepReport, b: SweepReport) -> SweepReport:
    """Associative, commutative merge (reference sweep.py:83-105)."""
    if (a.degree, a.fingerprint, a.raw_space) != (b.degree, b.fingerprint, b.raw_space):
        raise MergeMismatch("cannot merge reports over different triangulations or domains")
    hist = tuple(x + y for x, y in zip(a.oval_histogram, b.oval_histogram))
    schemes = dict(a.scheme_map)
    for s, (c, w) in b.scheme_map.items():
        if s in schemes:
            c0, w0 = schemes[s]
            schemes[s] = (c0 + c, min(w0, w))
        else:
            schemes[s] = (c, w)
    return SweepReport(a.degree, a.fingerprint, a.raw_space, hist, schemes,
                       a.total_classified + b.total_classified, {**a.params, **b.params})


def _domain_bits(d: int, raw_space: bool) -> int:
    bits = num_points(d) if raw_space else num_points(d) - 3
    if bits > _MAX_DOMAIN_BITS:
        raise BudgetExceeded(
            f"degree-{d} {'raw' if raw_space else 'representative'} space needs "
            f"{bits} index bits; at most {_MAX_DOMAIN_BITS} are supported"
        )
    return bits


def _classifier_for(T, classifier, device=None) -> Classifier:
    return classifier if classifier is not None else Classifier(T, device=device)


def report_from_agg(T, raw_space: bool, hist, total, keys, counts, wits, params) -> SweepReport:
    """Device aggregate -> SweepReport (strings rendered once per distinct key)."""
    d = T.degree
    nbins = harnack_bound(d) + 1
    if any(hist[nbins:]):
        raise InvariantViolation("oval histogram mass beyond the degree bound")
    odd = d % 2 == 1
    schemes = {
        scheme_from_key(int(k), odd): (int(c), int(w)) for k, c, w in zip(keys, counts, wits)
    }
    return SweepReport(d, fingerprint_of(T), raw_space, tuple(int(x) for x in hist[:nbins]),
                       schemes, int(total), params)


def _raise_status(rc: int, bad: int):
    raise InvariantViolation(f"{STATUS_MESSAGES.get(rc, f'status {rc}')} (at index {bad})")


def _run(T, c: Classifier, devices, fn_single, fn_multi):
    if devices and len(devices) > 1:
        plans = [c.native if dev == c.device else Classifier(T, device=dev).native
                 for dev in devices]
        return fn_multi(plans)
    return fn_single(c.native)


def sweep(T, sweep_range: SweepRange | None = None, workers: int = 1, raw_space: bool = False,
          chunk_size: int = DEFAULT_CHUNK, classifier: Classifier | None = None,
          devices: list[int] | None = None) -> SweepReport:
    """Classify every sign index in the range (default: the whole domain)."""
    bits = _domain_bits(T.degree, raw_space)
    domain = 1 << bits
    r = sweep_range or SweepRange(0, domain)
    if r.end > domain:
        raise IndexOutOfRange(f"sweep range end {r.end} exceeds domain size {domain}")
    c = _classifier_for(T, classifier, devices[0] if devices else None)
    rc, bad, agg = _run(
        T, c, devices,
        lambda p: p.sweep(raw_space, r.start, r.end),
        lambda plans: _lib.sweep_multi(plans, raw_space, r.start, r.end),
    )
    if rc:
        _raise_status(rc, bad)
    hist, total, keys, counts, wits = agg.result()
    params = {"mode": "sweep", "start": r.start, "end": r.end, "raw_space": raw_space}
    return report_from_agg(T, raw_space, hist, total, keys, counts, wits, params)


def sample(T, n: int, seed: int, workers: int = 1, chunk_size: int = DEFAULT_CHUNK,
           classifier: Classifier | None = None, devices: list[int] | None = None) -> SweepReport:
    """Classify n uniform draws from the representative space, reproducibly."""
    if n < 1:
        raise IndexOutOfRange(f"sample size must be positive, got {n}")
    nbits = _domain_bits(T.degree, raw_space=False)
    c = _classifier_for(T, classifier, devices[0] if devices else None)
    rc, bad, agg = _run(
        T, c, devices,
        lambda p: p.sample(seed, 0, n, nbits),
        lambda plans: _lib.sample_multi(plans, seed, 0, n, nbits),
    )
    if rc:
        _raise_status(rc, bad)
    hist, total, keys, counts, wits = agg.result()
    params = {"mode": "sample", "n": n, "seed": seed}
    return report_from_agg(T, False, hist, total, keys, counts, wits, params)


def sample_slice(T, seed: int, k0: int, k1: int, classifier: Classifier | None = None,
                 nbits: int | None = None) -> SweepReport:
    """Draws k0..k1-1 of the counter sampler (the reference's sample_kernel slice,
    kernels.py:447-462); partition-independent, so slices merge to ``sample``."""
    if not (0 <= k0 <= k1):
        raise IndexOutOfRange(f"bad draw range [{k0}, {k1})")
    nb = _domain_bits(T.degree, raw_space=False) if nbits is None else nbits
    c = _classifier_for(T, classifier)
    rc, bad, agg = c.native.sample(seed, k0, k1, nb)
    if rc:
        _raise_status(rc, bad)
    hist, total, keys, counts, wits = agg.result()
    params = {"mode": "sample-slice", "k0": k0, "k1": k1, "seed": seed}
    return report_from_agg(T, False, hist, total, keys, counts, wits, params)


def hist_array(report: SweepReport) -> np.ndarray:
    return np.asarray(report.oval_histogram, dtype=np.int64)
