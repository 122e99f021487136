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
_MAX_DOMAIN_BITS = 62  # indices must stay below 2^62 (reference sweep.py:32)


@dataclass(frozen=True)
class SweepRange:
    """Half-open index interval [start, end) of one enumeration domain."""

    start: int
    end: int

    def __post_init__(self):
        if self.start < 0 or self.end < self.start:
            raise IndexOutOfRange(f"bad sweep range [{self.start}, {self.end})")


@dataclass
class SweepReport:
    """Mergeable result of one enumeration (field contract: reference
    sweep.py:45-69).  ``scheme_map[s] = (count, witness)`` where the witness
    is the smallest index of the report's own domain classified as ``s``;
    ``params`` describe the run and take no part in equality."""

    degree: int
    fingerprint: str
    raw_space: bool
    oval_histogram: tuple[int, ...]
    scheme_map: dict[str, tuple[int, int]]
    total_classified: int
    params: dict = field(default_factory=dict, compare=False)

    def witness_bitstring(self, scheme: str) -> str:
        index = self.scheme_map[scheme][1]
        decode = sign_from_raw_index if self.raw_space else representative
        return decode(self.degree, index).bitstring()

    def distinct_schemes(self) -> int:
        return len(self.scheme_map)

    def max_ovals(self) -> int:
        nonzero = [k for k, c in enumerate(self.oval_histogram) if c]
        return nonzero[-1] if nonzero else 0


def empty_report(T, raw_space: bool = False) -> SweepReport:
    """The identity of :func:`merge` for T's domain."""
    bins = harnack_bound(T.degree) + 1
    return SweepReport(T.degree, fingerprint_of(T), raw_space, (0,) * bins, {}, 0)


def _merge_scheme_maps(x: dict, y: dict) -> dict:
    out = dict(x)
    for s, (cnt, wit) in y.items():
        have = out.get(s)
        out[s] = (cnt, wit) if have is None else (have[0] + cnt, min(have[1], wit))
    return out


def merge(a: SweepReport, b: SweepReport) -> SweepReport:
    """Associative, commutative combination: counts add, witnesses take the
    minimum, histograms add bin by bin (semantics of reference
    sweep.py:83-105; MergeMismatch on a different T or domain)."""
    ident_a = (a.degree, a.fingerprint, a.raw_space)
    if ident_a != (b.degree, b.fingerprint, b.raw_space):
        raise MergeMismatch("cannot merge reports over different triangulations or domains")
    hist = tuple(map(sum, zip(a.oval_histogram, b.oval_histogram)))
    params = dict(a.params)
    params.update(b.params)
    return SweepReport(*ident_a, hist, _merge_scheme_maps(a.scheme_map, b.scheme_map),
                       a.total_classified + b.total_classified, params)


def _domain_bits(d: int, raw_space: bool) -> int:
    """log2 of the domain size; BudgetExceeded beyond 62 bits."""
    bits = num_points(d) - (0 if raw_space else 3)
    if bits <= _MAX_DOMAIN_BITS:
        return bits
    kind = "raw" if raw_space else "representative"
    raise BudgetExceeded(f"degree-{d} {kind} space needs {bits} index bits; "
                         f"at most {_MAX_DOMAIN_BITS} are supported")


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
        return fn_multi(c.device_plans(devices))
    return fn_single(c.native)


def sweep(T, sweep_range: SweepRange | None = None, workers: int = 1, raw_space: bool = False,
          chunk_size: int = DEFAULT_CHUNK, classifier: Classifier | None = None,
          devices: list[int] | None = None) -> SweepReport:
    """Classify every sign index in the range (default: the whole domain)."""
    bits = _domain_bits(T.degree, raw_space)
    domain = 1 << bits
    r = sweep_range if sweep_range is not None else SweepRange(0, domain)
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
