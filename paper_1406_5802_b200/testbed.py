"""Trial engine for the paper's experiments on the B200 path (SURVEY.md §8(f),
rank 2): the reference's testbed (testbed/experiment.hpp, testbed/presets.hpp,
testbed/inputs.hpp) restated over this package's device-backed API, so the
Monte-Carlo tables run their solves and sketches on the GPU.

    run_experiment            experiment.hpp:30-69 (per-trial derived seeds,
                              failed trials counted, order-independent report;
                              trials run concurrently on a worker pool as the
                              reference's parallel_for_index does -- each
                              worker thread gets its own device context and
                              stream, so small trials overlap on the GPU)
    summarize                 stats.hpp:19-34
    gen_hard_block            inputs.hpp:18-49 (orthonormal_basis = CholeskyQR2,
                              which yields the same positive-diagonal Q as the
                              reference's Householder QR up to rounding)
    gen_lownumrank            inputs.hpp:67-83
    error_bounds_from_parts   lowrank.hpp:132-170 (the bound columns)
    run_hardblock_preprocessed  presets.hpp:90-119
    run_lowrank_preset        presets.hpp:121-179
    PRESETS                   every preset of presets.hpp:194-459 with the
                              reference's checks: table2 (GEPP baseline),
                              table3 (Gaussian), table4 (real circulant),
                              table5 (unitary circulant, complex pipeline),
                              table5a (DFT input, Gaussian rescue), table6 /
                              table7 (Gaussian sketch: rn1 / rn2), table8 /
                              table10 (real Toeplitz: rn2 / rn1), table9 /
                              table11 (unitary Toeplitz, complex: rn2 / rn1),
                              table12 (a-posteriori estimator), table13
                              (inverse-norm ratio), table14 (SRFT and
                              circulant-permutation sketch checks)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import randla as rl


# concurrent trial workers (each its own per-thread device context / stream)
WORKERS = 8


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
    slots = [None] * trials

    def one(t):
        try:
            slots[t] = run_trial(rl.derive_seed(seed, key, t), t)
        except rl.RandlaError:  # the reference catches std::runtime_error (types.hpp errors)
            slots[t] = None

    workers = min(trials, WORKERS)
    if workers <= 1:
        for t in range(trials):
            one(t)
    else:  # parallel_for_index (parallel.hpp:14-35): results land in per-trial slots
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(one, range(trials)))
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
                               refine: int, dims: Optional[List[int]] = None,
                               variant: rl.ToeplitzVariant = rl.ToeplitzVariant.REAL) -> List[ExperimentReport]:
    """presets.hpp:90-119: fresh hard-block input per trial, preprocess_solve with
    the multiplier seeded from the trial, one column per refinement stage; a
    complex family runs the complex pipeline on to_complex(a), to_complex(b)."""
    base = rl.MultiplierSpec(post_kind, 0, variant=variant)
    complex_path = rl.multiplier_is_complex(base)
    out = []
    for n in (dims if dims is not None else solve_dims(full)):
        def trial(ts, _t, n=n):
            a = gen_hard_block(n, rl.derive_seed(ts, 1))
            b = rl.gen_gaussian_vector(n, rl.derive_seed(ts, 2))
            post = rl.MultiplierSpec(post_kind, rl.derive_seed(ts, 3), variant=variant)
            if complex_path:
                a, b = rl.to_complex(a), rl.to_complex(b)
            hist = list(rl.preprocess_solve(a, b, None, post, refine).residual_history)
            while len(hist) < refine + 1:
                hist.append(hist[-1])
            return hist

        out.append(run_experiment(f"{label}/n={n}", trials, seed, [f"residual_iter{s}" for s in range(refine + 1)],
                                  trial, _TOKENS.get(post_kind, format_multiplier_token(base)), refine, n))
    return out


def run_dft_gaussian(seed: int, trials: int, full: bool, dims: Optional[List[int]] = None):
    """presets.hpp:254-284 (table5a): unpivoted elimination on the DFT matrix
    with a Gaussian rescue, one refinement step"""
    out = []
    for n in (dims if dims is not None else solve_dims(full)):
        a = rl.gen_dft_input(n)

        def trial(ts, _t, n=n, a=a):
            b = rl.to_complex(rl.gen_gaussian_vector(n, rl.derive_seed(ts, 2)))
            post = rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, rl.derive_seed(ts, 3))
            hist = list(rl.preprocess_solve(a, b, None, post, 1).residual_history)
            while len(hist) < 2:
                hist.append(hist[-1])
            return hist

        out.append(run_experiment(f"table5a/n={n}", trials, seed, ["residual_iter0", "residual_iter1"], trial,
                                  "gaussian", 1, n))
    return out


def run_posterior(seed: int, trials: int, full: bool, dims: Optional[List[int]] = None):
    """presets.hpp:344-378 (table12): the a-posteriori estimator (5 probes)
    against the true residual of the Gaussian zero-oversampling sketch"""
    out = []
    for n in (dims if dims is not None else lowrank_dims(full)):
        def trial(ts, _t, n=n):
            r = 8
            inst = gen_lownumrank(n, r, rl.derive_seed(ts, 1))
            spec = rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, rl.derive_seed(ts, 2))
            result = rl.range_find(inst.a, r, 0, spec, 0, with_residual=False)
            truth = rl.approximation_residual(inst.a, result)
            est = rl.posterior_estimate(inst.a, result, 5, rl.derive_seed(ts, 3))
            return [est, truth, 1.0 if est >= truth else 0.0]

        out.append(run_experiment(f"table12/n={n}", trials, seed, ["estimate", "true_rn2", "covered"], trial,
                                  "gaussian", 0, n))
    return out


def _check_table12(rs):
    c = CheckResult("estimate covers the true residual in >= 99% of trials at n=64")
    r = _report_at(rs, 64)
    if r is not None and r.column("covered").values:
        c.passed = r.column("covered").stats.mean >= 0.99
    return [c]


def run_srft_check(seed: int, trials: int, full: bool, dims: Optional[List[int]] = None):
    """presets.hpp:408-457 (table14): the sampled-transform sketch at its
    prescribed width against its guarantee, both variants"""
    out = []
    for n in (dims if dims is not None else ([64, 128, 256, 1024] if full else [64, 128])):
        for variant, vname in ((rl.SketchVariant.SRFT, "srft"), (rl.SketchVariant.CIRCULANT_PERMUTATION, "circperm")):
            def trial(ts, _t, n=n, variant=variant):
                r = 8
                inst = gen_lownumrank(n, r, rl.derive_seed(ts, 1))
                res = rl.srft_sketch_check(inst.a, r, rl.derive_seed(ts, 2), variant, inst.singulars[r])
                return [res.residual, res.bound, 1.0 if res.residual <= res.bound else 0.0]

            out.append(run_experiment(f"table14/{vname}/n={n}", trials, seed, ["residual", "bound", "within"], trial,
                                      vname, 0, n))
    return out


def lowrank_dims(full: bool) -> List[int]:
    """presets.hpp:39-41"""
    return [64, 128, 256, 512] if full else [64, 128]


def format_multiplier_token(spec) -> str:
    """multipliers.hpp:222-236"""
    k = rl.MultiplierKind(spec.kind)
    if k == rl.MultiplierKind.TOEPLITZ_BLOCK:
        return "toeplitz:variant=real" if spec.variant == rl.ToeplitzVariant.REAL else "toeplitz:variant=unitary"
    if k == rl.MultiplierKind.FINITE_SET_UNIFORM:
        return f"finite:card={spec.set_cardinality}"
    return {rl.MultiplierKind.NONE: "none", rl.MultiplierKind.GAUSSIAN: "gaussian",
            rl.MultiplierKind.REAL_CIRCULANT: "circulant", rl.MultiplierKind.UNITARY_CIRCULANT: "unitary-circulant",
            rl.MultiplierKind.SRFT: "srft", rl.MultiplierKind.CIRC_SKEW_PRODUCT: "circskew",
            rl.MultiplierKind.GAUSSIAN_CIRCULANT: "gaussian-circulant"}.get(k, "none")


@dataclass
class LowRankInstance:
    """inputs.hpp:60-65: the matrix and its construction's truncated factors"""
    a: np.ndarray
    left: np.ndarray      # truth.left (n x r)
    singulars: np.ndarray  # all n sigma_j
    right: np.ndarray     # truth.right (n x r)


def gen_lownumrank(n: int, r: int, seed: int) -> LowRankInstance:
    """inputs.hpp:67-83: sigma_j = 1/(j+1) up to r, 1e-10 beyond, between the
    orthonormal bases of two seeded Gaussians (CholeskyQR2 on the GPU)."""
    if r < 1 or r >= n:
        raise rl.DimensionError("gen_lownumrank: need 1 <= r < n")
    s = np.array(rl.orthonormal_basis(rl.gen_gaussian(n, n, rl.derive_seed(seed, 1))))
    t = np.array(rl.orthonormal_basis(rl.gen_gaussian(n, n, rl.derive_seed(seed, 2))))
    sigma = np.array([1.0 / (j + 1) if j < r else 1e-10 for j in range(n)])
    a = np.array(rl.matmul(s * sigma, np.ascontiguousarray(t.T)))
    return LowRankInstance(a, np.ascontiguousarray(s[:, :r]), sigma, np.ascontiguousarray(t[:, :r]))


@dataclass
class BoundReport:
    delta_plus: float = 0.0
    delta_plus_prime: float = 0.0
    sigma_r: float = 0.0
    sigma_r1: float = 0.0
    h_frobenius: float = 0.0
    t_h_inv_norm: float = 0.0


def error_bounds_from_parts(t_r, singulars, h, r) -> BoundReport:
    """lowrank.hpp:132-170 (the deterministic part): delta_plus =
    sqrt(2) ||H||_F ||(T_r^H H)^+|| sigma_{r+1} / sigma_r, delta_plus_prime =
    sigma_{r+1} + 2 delta_plus ||A||; T_r^H H and its singular values on the GPU."""
    if r < 1 or r > len(singulars):
        raise rl.DimensionError("error_bounds: rank out of range")
    rep = BoundReport(sigma_r=float(singulars[r - 1]), sigma_r1=float(singulars[r]) if r < len(singulars) else 0.0,
                      h_frobenius=float(np.linalg.norm(h)))
    gsv = rl.svd_values(rl.matmul(np.ascontiguousarray(t_r.conj().T), h))  # T_r^H H
    if not gsv[-1] > 0.0:
        raise rl.SingularMatrixError("unlucky multiplier: T_r^H H is singular, the bound is undefined")
    rep.t_h_inv_norm = 1.0 / gsv[-1]
    rep.delta_plus = math.sqrt(2.0) * rep.h_frobenius * rep.t_h_inv_norm * rep.sigma_r1 / rep.sigma_r
    rep.delta_plus_prime = rep.sigma_r1 + 2.0 * rep.delta_plus * float(singulars[0])
    return rep


def run_lowrank_preset(label: str, spec_base, basis_metric: bool, seed: int, trials: int, full: bool,
                       r: int = 8, dims: Optional[List[int]] = None) -> List[ExperimentReport]:
    """presets.hpp:121-179: zero-oversampling range finder on the known-rank
    inputs; rn1 (basis) or rn2 (approximation) and its ratio to the bound."""
    import copy
    out = []
    for n in (dims if dims is not None else lowrank_dims(full)):
        def trial(ts, _t, n=n):
            inst = gen_lownumrank(n, r, rl.derive_seed(ts, 1))
            spec = copy.copy(spec_base)
            spec.seed = rl.derive_seed(ts, 2)
            spec.rows, spec.cols = n, r
            if rl.multiplier_is_complex(spec):  # the complex pipeline on to_complex(a) (presets.hpp:150-160)
                ac = rl.to_complex(inst.a)
                result = rl.range_find(ac, r, 0, spec, 0)
                rep = error_bounds_from_parts(rl.to_complex(inst.right), inst.singulars, rl.materialize_complex(spec), r)
                if basis_metric:
                    rn, bound = rl.basis_residual(result, rl.to_complex(inst.left)), rep.delta_plus
                else:
                    rn, bound = rl.approximation_residual(ac, result), rep.delta_plus_prime
                return [rn, rn / bound]
            result = rl.range_find(inst.a, r, 0, spec, 0, with_residual=False)
            rep = error_bounds_from_parts(inst.right, inst.singulars, rl.materialize(spec), r)
            if basis_metric:
                rn, bound = rl.basis_residual(result, inst.left), rep.delta_plus
            else:
                rn, bound = rl.approximation_residual(inst.a, result), rep.delta_plus_prime
            return [rn, rn / bound]

        names = ["rn1", "ratio_rn1"] if basis_metric else ["rn2", "ratio_rn2"]
        out.append(run_experiment(f"{label}/n={n}", trials, seed, names, trial, format_multiplier_token(spec_base),
                                  0, n))
    return out


def run_gepp_baseline(seed: int, trials: int, full: bool, dims: Optional[List[int]] = None):
    """presets.hpp:195-219 (table2): pivoted elimination on the hard-block inputs"""
    out = []
    for n in (dims if dims is not None else solve_dims(full)):
        def trial(ts, _t, n=n):
            a = gen_hard_block(n, rl.derive_seed(ts, 1))
            b = rl.gen_gaussian_vector(n, rl.derive_seed(ts, 2))
            x = rl.lu_solve(rl.gepp_factor(a), b)  # solve_gepp (lu.hpp:150-153)
            return [float(np.linalg.norm(a @ x - b) / np.linalg.norm(b))]  # relative_residual (lu.hpp:155-161)
        out.append(run_experiment(f"table2/n={n}", trials, seed, ["residual"], trial, "none", 0, n))
    return out


def run_inverse_norm_ratio(seed: int, trials: int, full: bool, dims: Optional[List[int]] = None):
    """presets.hpp:380-406 (table13): ||(T_r^T H)^+|| against ||(H_rr)^+||"""
    out = []
    for n in (dims if dims is not None else lowrank_dims(full)):
        def trial(ts, _t, n=n):
            r = 8
            inst = gen_lownumrank(n, r, rl.derive_seed(ts, 1))
            h = rl.gen_gaussian(n, r, rl.derive_seed(ts, 2))
            num = 1.0 / rl.svd_values(rl.matmul(np.ascontiguousarray(inst.right.T), h))[-1]
            den = 1.0 / rl.svd_values(np.ascontiguousarray(h[:r, :r]))[-1]
            return [num / den]
        out.append(run_experiment(f"table13/n={n}", trials, seed, ["inv_norm_ratio"], trial, "gaussian", 0, n))
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


def check_fraction(reports, dim, column, threshold, quota) -> CheckResult:
    """presets.hpp:74-86: value <= threshold in >= quota of the trials (failed
    trials count against the quota)"""
    c = CheckResult(f"{column} <= {threshold:.3g} in >= {100 * quota:.3g}% of trials at n={dim}")
    r = _report_at(reports, dim)
    if r is None:
        return c
    hits = sum(1 for v in r.column(column).values if v <= threshold)
    c.passed = hits / r.trials >= quota
    return c


_G = rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN)
_TR = rl.MultiplierSpec(rl.MultiplierKind.TOEPLITZ_BLOCK, variant=rl.ToeplitzVariant.REAL)
_TU = rl.MultiplierSpec(rl.MultiplierKind.TOEPLITZ_BLOCK, variant=rl.ToeplitzVariant.UNITARY)


def _check_table14(rs):
    """presets.hpp:447-457: residual under the guarantee in >= 99% of trials, per report"""
    out = []
    for r in rs:
        col = r.column("within")
        out.append(CheckResult(f"{r.label}: residual under the guarantee in >= 99% of trials",
                               bool(col.values) and col.stats.mean >= 0.99))
    return out

PRESETS = {
    # presets.hpp:195-219
    "table2": (lambda seed, trials, full, dims=None: run_gepp_baseline(seed, trials, full, dims),
               lambda rs: [check_stat(rs, 64, "residual", False, 1e-11)]),
    # presets.hpp:221-232
    "table3": (lambda seed, trials, full, dims=None: run_hardblock_preprocessed(
                   "table3", rl.MultiplierKind.GAUSSIAN, seed, trials, full, 1, dims),
               lambda rs: [check_stat(rs, 64, "residual_iter0", True, 1e-4),
                           check_stat(rs, 64, "residual_iter0", False, 1e-6),
                           check_stat(rs, 64, "residual_iter1", False, 1e-11),
                           check_stat(rs, 128, "residual_iter1", False, 1e-11)]),
    # presets.hpp:234-242
    "table4": (lambda seed, trials, full, dims=None: run_hardblock_preprocessed(
                   "table4", rl.MultiplierKind.REAL_CIRCULANT, seed, trials, full, 1, dims),
               lambda rs: [check_stat(rs, 64, "residual_iter0", False, 1e-8)]),
    # presets.hpp:244-252: unitary circulant multipliers, the complex pipeline
    "table5": (lambda seed, trials, full, dims=None: run_hardblock_preprocessed(
                   "table5", rl.MultiplierKind.UNITARY_CIRCULANT, seed, trials, full, 1, dims),
               lambda rs: [check_stat(rs, 64, "residual_iter0", False, 1e-8)]),
    # presets.hpp:254-284: the DFT matrix with a Gaussian rescue
    "table5a": (lambda seed, trials, full, dims=None: run_dft_gaussian(seed, trials, full, dims),
                lambda rs: [check_fraction(rs, 256, "residual_iter0", 1e-4, 0.95)]),
    # presets.hpp:286-293
    "table6": (lambda seed, trials, full, dims=None: run_lowrank_preset("table6", _G, True, seed, trials, full,
                                                                         dims=dims),
               lambda rs: [check_fraction(rs, 64, "ratio_rn1", 1.01, 0.99)]),
    # presets.hpp:295-304
    "table7": (lambda seed, trials, full, dims=None: run_lowrank_preset("table7", _G, False, seed, trials, full,
                                                                         dims=dims),
               lambda rs: [check_stat(rs, 64, "rn2", False, 1e-6), check_stat(rs, 64, "ratio_rn2", False, 0.1),
                           check_fraction(rs, 64, "ratio_rn2", 1.0, 0.99)]),
    # presets.hpp:306-314
    "table8": (lambda seed, trials, full, dims=None: run_lowrank_preset("table8", _TR, False, seed, trials, full,
                                                                         dims=dims),
               lambda rs: [check_stat(rs, 64, "rn2", False, 1e-6), check_fraction(rs, 64, "ratio_rn2", 1.0, 0.99)]),
    # presets.hpp:316-324: unitary Toeplitz sketch (complex pipeline)
    "table9": (lambda seed, trials, full, dims=None: run_lowrank_preset("table9", _TU, False, seed, trials, full,
                                                                         dims=dims),
               lambda rs: [check_stat(rs, 64, "rn2", False, 1e-6), check_fraction(rs, 64, "ratio_rn2", 1.0, 0.99)]),
    # presets.hpp:326-333
    "table10": (lambda seed, trials, full, dims=None: run_lowrank_preset("table10", _TR, True, seed, trials, full,
                                                                          dims=dims),
                lambda rs: [check_fraction(rs, 64, "ratio_rn1", 1.01, 0.99)]),
    # presets.hpp:335-342: unitary Toeplitz sketch, basis residual
    "table11": (lambda seed, trials, full, dims=None: run_lowrank_preset("table11", _TU, True, seed, trials, full,
                                                                          dims=dims),
                lambda rs: [check_fraction(rs, 64, "ratio_rn1", 1.01, 0.99)]),
    # presets.hpp:408-457: the sampled-transform sketch against its guarantee
    "table14": (lambda seed, trials, full, dims=None: run_srft_check(seed, trials, full, dims),
                _check_table14),
    # presets.hpp:344-378: the a-posteriori estimator
    "table12": (lambda seed, trials, full, dims=None: run_posterior(seed, trials, full, dims), _check_table12),
    # presets.hpp:380-406 (no checks in the reference)
    "table13": (lambda seed, trials, full, dims=None: run_inverse_norm_ratio(seed, trials, full, dims),
                lambda rs: []),
}


def run_preset(name: str, seed: int, trials: int, full: bool = False, dims: Optional[List[int]] = None):
    """Run a preset and its checks: (reports, checks)."""
    run, check = PRESETS[name]
    reports = run(seed, trials, full, dims)
    return reports, check(reports)
