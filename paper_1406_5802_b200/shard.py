"""Multi-GPU decomposition of the batched path.

The batched 32x32 systems are independent (BASELINE config 2: system i uses
trial seed ts = base + i and the reference's per-trial derivation
A <- derive_seed(ts, 1), b <- derive_seed(ts, 2), G <- derive_seed(ts, 3),
testbed/presets.hpp:106-111), so the job shards by system index with no
data-path collective: rank r owns the contiguous block shard_bounds(total, r,
world) and generates exactly the seeds the single-process run would use for
those indices. The only exchange is the final per-batch summary (max growth,
max / summed residual, zero-pivot and counted systems), one all-reduce of a
few scalars.

The dense n=8192 solve does not shard (one LU, no 2D block-cyclic
decomposition): N GPUs run N independent replicas.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) block of `total` systems for `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if total < 0:
        raise ValueError("negative total")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def batch_seeds(lo: int, hi: int, base: int = 7) -> np.ndarray:
    """(hi - lo, 3) uint64 seeds for A, b, G of systems lo..hi-1
    (derive_seed(base + i, k), k = 1, 2, 3)."""
    from . import randla as _r
    return np.array([[_r.derive_seed(base + i, k) for k in (1, 2, 3)] for i in range(lo, hi)],
                    dtype=np.uint64).reshape(hi - lo, 3)


def local_summary(resid: np.ndarray, growth: np.ndarray, status: np.ndarray) -> dict:
    """Per-rank summary over the systems whose verdict passed (status 0)."""
    ok = np.asarray(status) == 0
    r = np.asarray(resid)[ok]
    g = np.asarray(growth)[ok]
    return {"max_growth": float(g.max()) if g.size else 0.0,
            "max_residual": float(r.max()) if r.size else 0.0,
            "sum_residual": float(r.sum()),
            "zero_pivots": int((~ok).sum()),
            "counted": int(ok.sum())}


def reduce_summary(local: dict, dist=None, device=None) -> dict:
    """All-reduce the per-rank summaries (max of maxima, sums of sums/counts).
    `dist` is torch.distributed (initialised) or None for one process;
    `device` is where the reduction tensors live ("cuda" for NCCL, cpu for gloo)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        out = dict(local)
    else:
        import torch
        mx = torch.tensor([local["max_growth"], local["max_residual"]], dtype=torch.float64, device=device)
        sm = torch.tensor([local["sum_residual"], float(local["zero_pivots"]), float(local["counted"])],
                          dtype=torch.float64, device=device)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        out = {"max_growth": float(mx[0]), "max_residual": float(mx[1]), "sum_residual": float(sm[0]),
               "zero_pivots": int(sm[1]), "counted": int(sm[2])}
    out["mean_residual"] = out["sum_residual"] / out["counted"] if out["counted"] else 0.0
    return out


def shard_inputs(lo: int, hi: int, base: int = 7):
    """(A, G, b) of systems lo..hi-1 as host arrays, from the reference's
    generators (bit-identical to the single-process inputs)."""
    from . import randla as _r
    seeds = batch_seeds(lo, hi, base)
    k = hi - lo
    a = _r.gen_gaussian_batch(k, 32, 32, seeds[:, 0])
    b = _r.gen_gaussian_batch(k, 32, 1, seeds[:, 1]).reshape(k, 32)
    g = _r.gen_gaussian_batch(k, 32, 32, seeds[:, 2])
    return a, g, b


def run_batched_shard(total: int, rank: int, world: int, dist=None, device=None, base: int = 7, solve=None,
                      to_device=None):
    """One rank's share of BASELINE config 2: its contiguous block of systems,
    generated from the per-trial seeds, solved by the library's batched entry
    point (randla.batched_preprocess_solve_32; `to_device` moves the inputs to
    the rank's GPU first), then the summary all-reduce. Returns
    (lo, hi, result, reduced summary)."""
    from . import randla as _r
    lo, hi = shard_bounds(total, rank, world)
    a, g, b = shard_inputs(lo, hi, base)
    if to_device is not None:
        a, g, b = to_device(a), to_device(g), to_device(b)
    out = (solve or _r.batched_preprocess_solve_32)(a, g, b)
    host = (lambda t: t) if isinstance(out.residual, np.ndarray) else (lambda t: t.cpu().numpy())
    local = local_summary(host(out.residual), host(out.growth), host(out.status))
    return lo, hi, out, reduce_summary(local, dist, device=device)
