"""Mergeable bivariate power-sum aggregates and histograms (host types).

Mirrors the aggregation part of the reference's ``lrcvt.stats``
(stats.py:19-221): ``MomentAggregate`` and its JSON form, ``merge``,
``comoment``, ``Histogram1D``/``Histogram2D``. The per-cell aggregation over a
tessellation runs on the GPU (``pipeline.aggregate_moments``); ``accumulate``
and ``histogram1d`` here are the reference's small-sample host utilities.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ORDERS = [(p, q) for p in range(5) for q in range(5) if p + q <= 4]


@dataclass
class MomentAggregate:
    """Raw power sums S_pq over one (x, y) pair, p + q <= 4 (stats.py:22-56)."""

    x_name: str = "x"
    y_name: str = "y"
    n: int = 0
    sums: np.ndarray = field(default_factory=lambda: np.zeros((5, 5)))
    min_x: float = math.inf
    max_x: float = -math.inf
    min_y: float = math.inf
    max_y: float = -math.inf

    def variable_pair(self) -> tuple[str, str]:
        return (self.x_name, self.y_name)

    def to_dict(self) -> dict:
        return {
            "x": self.x_name,
            "y": self.y_name,
            "n": int(self.n),
            "sums": {f"{p},{q}": float(self.sums[p, q]) for p, q in ORDERS},
            "min": [self.min_x, self.min_y],
            "max": [self.max_x, self.max_y],
        }

    @classmethod
    def from_dict(cls, d: dict) -> "MomentAggregate":
        agg = cls(x_name=d["x"], y_name=d["y"], n=int(d["n"]))
        for key, val in d["sums"].items():
            p, q = (int(t) for t in key.split(","))
            agg.sums[p, q] = val
        agg.min_x, agg.min_y = d["min"]
        agg.max_x, agg.max_y = d["max"]
        return agg


def accumulate(samples, x_name: str = "x", y_name: str = "y") -> MomentAggregate:
    """Exactly rounded power sums of explicit samples (stats.py:59-78)."""
    samples = np.asarray(samples, dtype=np.float64).reshape(-1, 2)
    if samples.size and not np.isfinite(samples).all():
        raise ValueError("samples must be finite")
    agg = MomentAggregate(x_name=x_name, y_name=y_name, n=samples.shape[0])
    if samples.shape[0] == 0:
        return agg
    x, y = samples[:, 0], samples[:, 1]
    xp = [np.ones_like(x), x, x * x, x**3, x**4]
    yq = [np.ones_like(y), y, y * y, y**3, y**4]
    for p, q in ORDERS:
        agg.sums[p, q] = math.fsum(xp[p] * yq[q])
    agg.min_x, agg.max_x = float(x.min()), float(x.max())
    agg.min_y, agg.max_y = float(y.min()), float(y.max())
    return agg


def merge(a: MomentAggregate, b: MomentAggregate) -> MomentAggregate:
    """Combine two aggregates of the same pair (stats.py:81-94)."""
    if a.variable_pair() != b.variable_pair():
        raise ValueError(f"variable pair mismatch: {a.variable_pair()} vs {b.variable_pair()}")
    out = MomentAggregate(x_name=a.x_name, y_name=a.y_name, n=a.n + b.n)
    out.sums = a.sums + b.sums
    out.min_x = min(a.min_x, b.min_x)
    out.max_x = max(a.max_x, b.max_x)
    out.min_y = min(a.min_y, b.min_y)
    out.max_y = max(a.max_y, b.max_y)
    return out


def comoment(agg: MomentAggregate, p: int, q: int) -> float:
    """Central co-moment E[(x-mx)^p (y-my)^q] by binomial expansion (stats.py:97-116)."""
    if agg.n < 1:
        raise ValueError("empty aggregate has no moments")
    if p + q > 4 or p < 0 or q < 0:
        raise ValueError(f"order ({p},{q}) out of range (p+q <= 4)")
    n = agg.n
    mx = agg.sums[1, 0] / n
    my = agg.sums[0, 1] / n
    total = 0.0
    for i in range(p + 1):
        for j in range(q + 1):
            total += math.comb(p, i) * math.comb(q, j) * (-mx) ** (p - i) * (-my) ** (q - j) * agg.sums[i, j]
    return total / n


def mean_xy(agg: MomentAggregate) -> tuple[float, float]:
    if agg.n < 1:
        raise ValueError("empty aggregate has no mean")
    return (agg.sums[1, 0] / agg.n, agg.sums[0, 1] / agg.n)


@dataclass
class Histogram1D:
    lo: float
    hi: float
    counts: np.ndarray
    underflow: int = 0
    overflow: int = 0

    @property
    def n(self) -> int:
        return int(self.counts.sum()) + self.underflow + self.overflow

    def centers(self) -> np.ndarray:
        edges = np.linspace(self.lo, self.hi, self.counts.size + 1)
        return 0.5 * (edges[:-1] + edges[1:])

    def merge(self, other: "Histogram1D") -> "Histogram1D":
        if (self.lo, self.hi, self.counts.size) != (other.lo, other.hi, other.counts.size):
            raise ValueError("histogram axes differ; cannot merge")
        return Histogram1D(self.lo, self.hi, self.counts + other.counts,
                           self.underflow + other.underflow, self.overflow + other.overflow)


@dataclass
class Histogram2D:
    x_lo: float
    x_hi: float
    y_lo: float
    y_hi: float
    counts: np.ndarray
    out_of_range: int = 0

    @property
    def n(self) -> int:
        return int(self.counts.sum()) + self.out_of_range

    def centers(self):
        ex = np.linspace(self.x_lo, self.x_hi, self.counts.shape[0] + 1)
        ey = np.linspace(self.y_lo, self.y_hi, self.counts.shape[1] + 1)
        return 0.5 * (ex[:-1] + ex[1:]), 0.5 * (ey[:-1] + ey[1:])

    def merge(self, other: "Histogram2D") -> "Histogram2D":
        same = ((self.x_lo, self.x_hi, self.y_lo, self.y_hi) == (other.x_lo, other.x_hi, other.y_lo, other.y_hi)
                and self.counts.shape == other.counts.shape)
        if not same:
            raise ValueError("histogram axes differ; cannot merge")
        return Histogram2D(self.x_lo, self.x_hi, self.y_lo, self.y_hi, self.counts + other.counts,
                           self.out_of_range + other.out_of_range)


def axis_range(values, lo=None, hi=None):
    """stats.py:186-191: data range unless given; empty span widened by 1."""
    lo = float(values.min()) if lo is None else float(lo)
    hi = float(values.max()) if hi is None else float(hi)
    if hi <= lo:
        hi = lo + 1.0
    return lo, hi


def histogram1d(values, bins=64, lo=None, hi=None) -> Histogram1D:
    values = np.asarray(values, dtype=np.float64).ravel()
    lo, hi = axis_range(values, lo, hi)
    inside = (values >= lo) & (values <= hi)
    counts, _ = np.histogram(values[inside], bins=bins, range=(lo, hi))
    return Histogram1D(lo, hi, counts.astype(np.int64), underflow=int(np.count_nonzero(values < lo)),
                       overflow=int(np.count_nonzero(values > hi)))


def histogram2d(samples, bins=(48, 48), x_range=None, y_range=None) -> Histogram2D:
    samples = np.asarray(samples, dtype=np.float64).reshape(-1, 2)
    x_lo, x_hi = axis_range(samples[:, 0], *(x_range or (None, None)))
    y_lo, y_hi = axis_range(samples[:, 1], *(y_range or (None, None)))
    inside = ((samples[:, 0] >= x_lo) & (samples[:, 0] <= x_hi)
              & (samples[:, 1] >= y_lo) & (samples[:, 1] <= y_hi))
    counts, _, _ = np.histogram2d(samples[inside, 0], samples[inside, 1], bins=bins,
                                  range=((x_lo, x_hi), (y_lo, y_hi)))
    return Histogram2D(x_lo, x_hi, y_lo, y_hi, counts.astype(np.int64),
                       out_of_range=int(np.count_nonzero(~inside)))
