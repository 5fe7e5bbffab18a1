"""Trial engine for the paper's preprocessed-GENP experiments on the B200 path
(SURVEY.md §8(f), rank 2): the reference's testbed (testbed/experiment.hpp,
testbed/presets.hpp, testbed/inputs.hpp) restated over this package's
device-backed API, so the Monte-Carlo tables run their solves on the GPU.

    run_experiment            experiment.hpp:30-69 (per-trial derived seeds,
                              failed trials counted, order-independent report)
    summarize                 stats.hpp:19-34
    gen_hard_block            inputs.hpp:18-49 (orthonormal_basis = CholeskyQR2,
                              which yields the same positive-diagonal Q as the
                              reference's Householder QR up to rounding)
    run_hardblock_preprocessed  presets.hpp:90-119
    PRESETS                   table3 (Gaussian) and table4 (real circulant)
                              with the reference's checks (presets.hpp:219-240)

Complex families (table5, table5a) are outside this path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import randla as rl


@dataclass
class StatSummary:
    mean: float = 0.0
    max: float = 0.0
    min: float = 0.0
    std: float = 0.0


def summarize(values) -> StatSummary:
    """stats.hpp:19-34: sequential sum, population standard deviation."""
    if len(values) == 0:
        raise ValueError("summarize: no values")
    s = StatSummary(min=values[0], max=values[0])
    total = 0.0
    for v in values:
        total += v
        s.min = min(s.min, v)
        s.max = max(s.max, v)
    s.mean = total / len(values)
    var = 0.0
    for v in values:
        var += (v - s.mean) * (v - s.mean)
    s.std = math.sqrt(var / len(values))
    return s


@dataclass
class ReportColumn:
    name: str
    stats: StatSummary = field(default_factory=StatSummary)
    values: List[float] = field(default_factory=list)


@dataclass
class ExperimentReport:
    label: str
    trials: int = 0
    failures: int = 0
    columns: List[ReportColumn] = field(default_factory=list)
    seed: int = 0
    multiplier: str = "none"
    refine_steps: int = 0
    dimension: int = 0

    def column(self, name: str) -> ReportColumn:
        for c in self.columns:
            if c.name == name:
                return c
        raise KeyError(name)


def run_experiment(label: str, trials: int, seed: int, metric_names: List[str],
                   run_trial: Callable[[int, int], Optional[List[float]]], multiplier: str = "none",
                   refine_steps: int = 0, dimension: int = 0) -> ExperimentReport:
    """experiment.hpp:30-69: trial t runs with derive_seed(seed, hash_label(label), t);
    a trial that raises a runtime error (ZeroPivotError, ...) counts as a failure."""
    if trials < 1:
        raise rl.DimensionError("run_experiment: trials must be >= 1")
    key = rl.hash_label(label)
    slots = []
    for t in range(trials):
        try:
            slots.append(run_trial(rl.derive_seed(seed, key, t), t))
        except rl.RandlaError:  # the reference catches std::runtime_error (types.hpp errors)
            slots.append(None)
    rep = ExperimentReport(label=label, trials=trials, seed=seed, multiplier=multiplier, refine_steps=refine_steps,
                           dimension=dimension)
    cols = [[] for _ in metric_names]
    for slot in slots:
        if slot is None:
            rep.failures += 1
            continue
        if len(slot) != len(metric_names):
            raise rl.LogicError("trial produced wrong metric count")
        for c, v in enumerate(slot):
            cols[c].append(float(v))
    for name, vals in zip(metric_names, cols):
        col = ReportColumn(name=name, values=vals)
        if vals:
            col.stats = summarize(vals)
        rep.columns.append(col)
    return rep


def gen_hard_block(n: int, seed: int) -> np.ndarray:
    """inputs.hpp:18-49: leading n/2 block U diag(1, .., 1, 0, 0, 0, 0) V^T (exactly
    four zero singular values) bordered by Gaussian Toeplitz blocks rescaled to
    unit spectral-norm estimate. Products, bases and norms run on the GPU."""
    if n < 8 or n % 2 != 0:
        raise rl.DimensionError("gen_hard_block: need even n >= 8")
    k = n // 2
    u = np.array(rl.orthonormal_basis(rl.gen_gaussian(k, k, rl.derive_seed(seed, 1))))
    v = np.array(rl.orthonormal_basis(rl.gen_gaussian(k, k, rl.derive_seed(seed, 2))))
    u[:, k - 4:] = 0.0
    a_k = np.array(rl.matmul(u, np.ascontiguousarray(v.T)))

    def toeplitz(s):
        d = rl.gen_gaussian_vector(2 * k - 1, s)  # RngStream(s).next_gaussian() x (2k - 1)
        i = np.arange(k)
        t = d[(i[:, None] + (k - 1)) - i[None, :]]
        return t / rl.spectral_norm_estimate(t)

    out = np.empty((n, n))
    out[:k, :k] = a_k
    out[:k, k:] = toeplitz(rl.derive_seed(seed, 3))
    out[k:, :k] = toeplitz(rl.derive_seed(seed, 4))
    out[k:, k:] = toeplitz(rl.derive_seed(seed, 5))
    return out


def solve_dims(full: bool) -> List[int]:
    """presets.hpp:35-37"""
    return [64, 128, 256, 512, 1024] if full else [64, 128, 256]


_TOKENS = {rl.MultiplierKind.GAUSSIAN: "gaussian", rl.MultiplierKind.REAL_CIRCULANT: "real_circulant",
           rl.MultiplierKind.GAUSSIAN_CIRCULANT: "gaussian_circulant"}


def run_hardblock_preprocessed(label: str, post_kind: rl.MultiplierKind, seed: int, trials: int, full: bool,
                               refine: int, dims: Optional[List[int]] = None) -> List[ExperimentReport]:
    """presets.hpp:90-119: fresh hard-block input per trial, preprocess_solve with
    the multiplier seeded from the trial, one column per refinement stage."""
    out = []
    for n in (dims if dims is not None else solve_dims(full)):
        def trial(ts, _t, n=n):
            a = gen_hard_block(n, rl.derive_seed(ts, 1))
            b = rl.gen_gaussian_vector(n, rl.derive_seed(ts, 2))
            post = rl.MultiplierSpec(post_kind, rl.derive_seed(ts, 3))
            hist = list(rl.preprocess_solve(a, b, None, post, refine).residual_history)
            while len(hist) < refine + 1:
                hist.append(hist[-1])
            return hist

        out.append(run_experiment(f"{label}/n={n}", trials, seed, [f"residual_iter{s}" for s in range(refine + 1)],
                                  trial, _TOKENS.get(post_kind, "none"), refine, n))
    return out


@dataclass
class CheckResult:
    description: str
    passed: bool = False


def _report_at(reports, dim):
    for r in reports:
        if r.dimension == dim:
            return r
    return None


def check_stat(reports, dim, column, use_max, threshold) -> CheckResult:
    """presets.hpp:58-72"""
    c = CheckResult(f"{'max' if use_max else 'mean'} {column} <= {threshold:.3g} at n={dim}")
    r = _report_at(reports, dim)
    if r is None:
        return c
    col = r.column(column)
    if not col.values:
        return c
    c.passed = (col.stats.max if use_max else col.stats.mean) <= threshold
    return c


PRESETS = {
    # presets.hpp:219-233
    "table3": (lambda seed, trials, full, dims=None: run_hardblock_preprocessed(
                   "table3", rl.MultiplierKind.GAUSSIAN, seed, trials, full, 1, dims),
               lambda rs: [check_stat(rs, 64, "residual_iter0", True, 1e-4),
                           check_stat(rs, 64, "residual_iter0", False, 1e-6),
                           check_stat(rs, 64, "residual_iter1", False, 1e-11),
                           check_stat(rs, 128, "residual_iter1", False, 1e-11)]),
    # presets.hpp:235-243
    "table4": (lambda seed, trials, full, dims=None: run_hardblock_preprocessed(
                   "table4", rl.MultiplierKind.REAL_CIRCULANT, seed, trials, full, 1, dims),
               lambda rs: [check_stat(rs, 64, "residual_iter0", False, 1e-8)]),
}


def run_preset(name: str, seed: int, trials: int, full: bool = False, dims: Optional[List[int]] = None):
    """Run a preset and its checks: (reports, checks)."""
    run, check = PRESETS[name]
    reports = run(seed, trials, full, dims)
    return reports, check(reports)
