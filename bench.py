#!/usr/bin/env python
"""Benchmark driver (one JSON line on rank 0).

Workload (BASELINE.json metric "preprocessed-GENP FP64 TFLOP/s at n=8192, % of
FP64 peak; batched solves/s"): one step = one Gaussian-preprocessed GENP
solve at n=8192 — preprocess_solve(A, b, none, {Gaussian, G}, 0)
(preprocess.hpp:156-180): product A*G, blocked GENP with the pivot verdict,
chain solve x = G (LU)^-1 b — with A (seed 1), G (seed 2), b (seed 3) resident
in HBM. value = F(n) / step time in TFLOP/s, F(n) = (2n^3 - n^2) +
sum_{m<n} m(1+2m) + 2n^2 + (2n^2 - n). The batched-32 figure
(BASELINE config 2, 65,536 systems) rides along under "secondary", and
configs 3-5 under "configs_3_to_5" on the inputs of tools/config_inputs.py
(the bytes the reference-made fixtures in tests/golden/ were computed on).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--gpus N > 1 without a torchrun environment relaunches itself under
torch.distributed.run (one process per GPU, NCCL, 127.0.0.1). The dense
solve does not shard (replicas); the batched systems shard by
index. --dry-run exercises the launcher and the collectives (gloo) without a
GPU and prints the line's n_gpus.

--impl reference times the reference's own CPU implementation of the same
workload: oracle/_ref (the reference headers compiled from /root/reference)
runs one full n = 8192 preprocess_solve per host core concurrently on the
reference's parallel_for_index pool; one such step is several minutes of CPU,
so the arm times exactly one step after no warm-up whatever --steps/--warmup
say (the line records it).
"""
import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

METRIC = "preprocessed-GENP FP64 TFLOP/s at n=8192, % of FP64 peak; batched solves/s"
FP64_PEAK_TFLOPS = 35.46   # cuBLAS DGEMM 8192^3 measured on this pool's B200 (profiles/r01_fp64_peak.txt)


def profiled_traffic(name, systems=None):
    """dram__bytes_read + dram__bytes_write per launch of a kernel, from the
    newest committed ncu --set full capture (profiles/rNN_<name>_traffic.json,
    written by tools/write_profiles.py); scaled to `systems` for the batched
    kernel. None when no capture is committed."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r[0-9][0-9]_{name}_traffic.json")))
    if not paths:
        return None
    try:
        d = json.load(open(paths[-1]))
        t = d.get("dram_bytes_per_launch")
        if t is not None and systems is not None and d.get("systems"):
            t = t * systems / d["systems"]
        return t
    except Exception:
        return None
FP64_DMMA_PEAK = 37.06     # DMMA issue-rate microbenchmark (tools/fp64_peak.cu)
BATCH_BYTES_PER_SYSTEM = 25104
WORKLOAD = "Gaussian-preprocessed GENP solve, n=8192 (BASELINE headline; config 1 recipe at n=8192)"


def flops_dense(n):
    """F(n) of SURVEY §8(d)."""
    return (2 * n ** 3 - n ** 2) + sum_lu_flops(n) + 2 * n ** 2 + (2 * n ** 2 - n)


def sum_lu_flops(n):
    return n * (n - 1) // 2 + 2 * ((n - 1) * n * (2 * n - 1) // 6)


def lu_step_flops(n, j0, j1):
    """flops of elimination steps j0..j1-1 of genp_factor: (n-1-j)(1 + 2(n-1-j))"""
    return sum((n - 1 - j) * (1 + 2 * (n - 1 - j)) for j in range(j0, min(j1, n)))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def base_config(n, world):
    return {"workload": WORKLOAD, "n": n, "refine_steps": 0, "multiplier": "gaussian",
            "l2": "inputs 1 GiB per step > 126 MB L2 (no flush needed)",
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}


# ---- clocks during the timed region ---------------------------------------
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sync_boost", 0x40: "sw_thermal_slowdown", 0x80: "hw_thermal_slowdown",
               0x100: "hw_power_brake_slowdown", 0x200: "display_clock_setting"}


class ClockSampler:
    def __init__(self, gpu_index):
        self.gpu = str(gpu_index)
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu, "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out = self.proc.communicate()[0]
        sm, mx, reasons = [], [], set()
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[3], 16)
            except ValueError:
                continue
            for b, name in REASON_BITS.items():
                if bits & b and b != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- distributed plumbing ----------------------------------------------------
def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Dist:
    def __init__(self, world, local, backend="nccl"):
        import torch
        self.torch = torch
        self.world = world
        self.device = "cuda" if backend == "nccl" else "cpu"
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if backend == "nccl":
                torch.cuda.set_device(local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group("gloo")
            self.dist = dist
        else:
            self.dist = None

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, v):
        if not self.dist:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# ---- the reference's CPU path ------------------------------------------------------
def reference_full(n, trials):
    """The reference's own code (oracle/_ref) on the headline workload:
    `trials` concurrent preprocess_solve(A, b, none, {Gaussian, 2}, 0) at n on
    the reference's parallel_for_index pool (A, b of the headline; G drawn
    inside from seed 2, as the reference does). Returns (seconds, info)."""
    import oracle
    if oracle.REF is None:
        raise RuntimeError("oracle/_ref not built")
    a = oracle.REF.gen_gaussian(n, n, 1)
    b = oracle.REF.gen_gaussian(n, 1, 3).reshape(n)
    a_all = np.empty((trials, n, n))
    a_all[:] = a
    b_all = np.empty((trials, n))
    b_all[:] = b
    seeds = np.full(trials, 2, dtype=np.uint64)
    t0 = time.perf_counter()
    res, nf = oracle.REF.parallel_dense_trials(a_all, b_all, seeds)
    dt = time.perf_counter() - t0
    return dt, {"kind": "reference", "cores": trials, "zero_pivots": nf, "median_residual": float(np.nanmedian(res)),
                "sample": f"{trials} concurrent full preprocess_solve(A, b, none, {{Gaussian, 2}}, 0) at n={n} "
                          f"(the headline workload itself) on the reference's parallel_for_index pool, one step"}


def port_sample(n, threads, rows=64, steps=48):
    """Bounded sample of the headline workload on the host cores with the
    oracle's line-cited restatement (kind "port"; bit-identical to the
    reference's genp_factor, tests/test_oracle.py): per thread, the product
    rows [t R, (t+1) R) of A*G by the single-thread GEMM hook (the reference's
    Eigen product is single-threaded) and the first `steps` elimination steps
    of genp_factor on a full n x n matrix (the same memory traffic per step as
    the whole factorisation's early steps). TFLOP/s = sampled flops / wall."""
    import oracle
    C = oracle.C
    a = C.gen_gaussian(n, n, 1)
    g = C.gen_gaussian(n, n, 2)
    mats = [np.array(a) for _ in range(threads)]  # untimed copies: each thread eliminates its own matrix
    flops = [0] * threads

    def work(t):
        r0 = (t * rows) % n
        C.matmul(a[r0:r0 + rows], g)
        C.genp_steps(mats[t], 0, steps)
        flops[t] = 2 * rows * n * n + lu_step_flops(n, 0, steps)

    th = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    t0 = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    dt = time.perf_counter() - t0
    tf = sum(flops) / dt / 1e12
    return tf, {"kind": "port", "cores": threads, "seconds": dt,
                "sample": f"bounded sample of the n={n} headline workload on {threads} threads: per thread "
                          f"{rows} product rows of A*G (single-thread GEMM, as the reference's Eigen) + the first "
                          f"{steps} elimination steps of genp_factor on a full {n}x{n} matrix (oracle/oracle.c "
                          f"restatement, bit-identical to the reference's loop); TFLOP/s = sampled flops / wall"}


def run_reference(args):
    rank, world, local = dist_info()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    n = args.n
    dt, info = reference_full(n, cores)
    tf = cores * flops_dense(n) / dt / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": tf, "unit": "TFLOP/s", "n_gpus": 0, "steps": 1,
            "warmup": 0, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic: exact reference RNG, A=gen_gaussian(n,n,1), G=gen_gaussian(n,n,2), "
                                    "b=gen_gaussian_vector(n,3)",
            "config": base_config(n, 1),
            "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": info["kind"],
                             "sample": info["sample"]},
            "e2e": {"value": tf, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "median_residual": info["median_residual"], "zero_pivots": info["zero_pivots"]}
    print(json.dumps(line), flush=True)
    return 0


# ---- BASELINE configs 3-5 on the fixture inputs -------------------------------------
def measure_configs_3_to_5(rl, capi, L, torch, stream, hbm):
    """Config 3: circulant-preprocessed GENP at n=8192 (FFT product + blocked
    GENP + FFT chain solve); config 4: range finder m=n=8192, r=64, Gaussian H;
    config 5: m=32768, n=16384, r=256, Toeplitz H by FFT. Inputs: the pinned
    deterministic build of tools/config_inputs.py (the bytes of the
    reference-made fixtures, SHA-256 in the line), untimed."""
    import config_inputs
    out = {}
    work = tempfile.mkdtemp(prefix="randla_bench_inputs_")

    def ev_time(f, reps=1):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            f()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    def load(cfg):
        rec = config_inputs.build(cfg, work)
        inp = config_inputs.load(cfg, work)
        dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items() if k != "record"}
        for k in ("A", "b", "c"):
            p = os.path.join(work, f"{cfg}_{k}.npy")
            if os.path.exists(p):
                os.remove(p)
        return rec["sha256"], dev

    # ---- config 3
    n = 8192
    sha, d = load("cfg3")
    a, b, c = d["A"], d["b"], d["c"]
    x = torch.empty_like(b)
    ac = torch.empty_like(a)
    fft_ms = ev_time(lambda: L.rl_circulant_right_multiply(None, capi.RL_DEVICE, n, n, a.data_ptr(), c.data_ptr(),
                                                           ac.data_ptr()), 3)
    del ac
    m3 = capi.rl_multiplier()
    m3.kind = capi.RL_MULT_GAUSSIAN_CIRCULANT
    m3.column = c.data_ptr()
    info = capi.rl_solve_info()

    def solve3():
        rc = L.rl_preprocessed_genp_solve(None, capi.RL_DEVICE, n, a.data_ptr(), b.data_ptr(), None, ctypes.byref(m3),
                                          0, x.data_ptr(), None, 0, ctypes.byref(info))
        if rc != 0:
            raise RuntimeError(capi.last_error())
    ms3 = ev_time(solve3, 2)
    fft_bytes = 2 * 8 * n * n
    out["config3"] = {
        "workload": "circulant-preprocessed GENP, n=8192, kappa=1e4 (Haar U/V seeds 11/12), Gaussian circulant "
                    "seed 13, b seed 14", "inputs_sha256": sha,
        "ms_per_call": ms3, "stage_ms": list(info.stage_ms), "residual_b": info.residual_history[0],
        "growth": info.growth,
        "fft_product": {"ms": fft_ms, "roofline": {"bound": "hbm", "achieved": fft_bytes / (fft_ms * 1e-3) / 1e9,
                                                    "peak": hbm, "unit": "GB/s",
                                                    "frac": fft_bytes / (fft_ms * 1e-3) / 1e9 / hbm,
                                                    "algorithmic_bytes": fft_bytes}},
        "lu_tflops": sum_lu_flops(n) / (info.stage_ms[1] * 1e-3) / 1e12}
    del a, b, c, x, d

    # ---- config 4
    sha, d = load("cfg4")
    a = d["A"]
    m, n = a.shape
    r = 64
    out["config4"] = run_range_find(L, capi, a, r, capi.RL_MULT_GAUSSIAN, 41, ev_time, 3 * 2 * m * n * r,
                                    "range finder m=n=8192, r=64, Gaussian H (seed 41); sigma 1..1e-2, "
                                    "E = 1e-10 gen_gaussian(seed 44)")
    out["config4"]["inputs_sha256"] = sha
    del a, d

    # ---- config 5
    sha, d = load("cfg5")
    a = d["A"]
    m, n = a.shape
    r = 256
    res5 = run_range_find(L, capi, a, r, capi.RL_MULT_GAUSSIAN_CIRCULANT, 21, ev_time, 2 * 2 * m * n * r,
                          "range finder m=32768, n=16384, r=256, Toeplitz H (Gaussian circulant seed 21); "
                          "sigma 1..1e-3, E = 1e-12 gen_gaussian(seed 53)")
    res5["inputs_sha256"] = sha
    cc = d["c"]
    y = torch.empty(m, r, dtype=torch.float64, device="cuda")
    sk_ms = ev_time(lambda: L.rl_toeplitz_right_multiply(None, capi.RL_DEVICE, m, n, a.data_ptr(), n, cc.data_ptr(), r,
                                                         y.data_ptr()), 3)
    sk_bytes = 8 * m * n + 8 * m * r
    res5["toeplitz_sketch"] = {"ms": sk_ms, "roofline": {"bound": "hbm", "achieved": sk_bytes / (sk_ms * 1e-3) / 1e9,
                                                         "peak": hbm, "unit": "GB/s",
                                                         "frac": sk_bytes / (sk_ms * 1e-3) / 1e9 / hbm,
                                                         "algorithmic_bytes": sk_bytes}}
    out["config5"] = res5
    del a, y, d
    torch.cuda.empty_cache()
    return out


def run_range_find(L, capi, a, r, kind, seed, ev_time, gemm_flops, workload):
    m, n = a.shape
    q = a.new_empty(m, r)
    mlt = capi.rl_multiplier()
    mlt.kind = kind
    mlt.seed = seed
    info = capi.rl_lowrank_info()

    def call():
        rc = L.rl_range_find_residual(None, capi.RL_DEVICE, m, n, a.data_ptr(), r, ctypes.byref(mlt), 0, q.data_ptr(),
                                      ctypes.byref(info))
        if rc != 0:
            raise RuntimeError(capi.last_error())
    ms = ev_time(call, 1)
    return {"workload": workload, "ms_per_call": ms, "residual_frobenius": info.residual_frobenius,
            "residual_spectral": info.residual_spectral, "power_iterations": info.power_iterations,
            "product_tflops_equiv": gemm_flops / (ms * 1e-3) / 1e12,
            "note": "call = sketch + CholeskyQR2 + Q^T A + residual ||.||_F + power-iteration ||.||_2"}


# ---- end to end through the public APIs ------------------------------------------
def e2e_python(rl, torch, A, b, n, steps, D, world, ref_x):
    """rl.preprocess_solve on pinned host numpy buffers (the Python public API):
    every step uploads A and b, draws G from seed 2 on the device, factors,
    solves and returns x on the host."""
    hA = torch.from_numpy(A).pin_memory()
    hb = torch.from_numpy(b).pin_memory()
    a_np, b_np = hA.numpy(), hb.numpy()
    spec = rl.MultiplierSpec(rl.MultiplierKind.GAUSSIAN, 2)
    out = rl.preprocess_solve(a_np, b_np, None, spec, 0)
    D.barrier()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        out = rl.preprocess_solve(a_np, b_np, None, spec, 0)
        ts.append(time.perf_counter() - t0)
    t = D.max(statistics.mean(ts))
    F = flops_dense(n)
    return {"value": world * F / t / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 8 * n * n + 8 * n,
            "d2h_bytes_per_step": 8 * n, "ms_per_step": t * 1e3, "steps": steps,
            "api": "paper_1406_5802_b200.preprocess_solve(A, b, None, MultiplierSpec(GAUSSIAN, 2), 0), pinned numpy",
            "includes": "H2D of A (4 row blocks on a side stream, overlapped with the product) and b from pinned "
                        "memory, exact generation of G from seed 2 on the device (the ~6% of log evaluations "
                        "glibc must decide finished on the host), product, GENP, verdict, solve, D2H of x",
            "matches_device_resident_x": bool(np.array_equal(out.x, ref_x))}


def e2e_cpp_header(n, steps):
    """tools/_build/e2e_header: the C++ drop-in header's preprocess_solve on
    RealMatrix / std::vector (pageable host memory), as a reference user calls it."""
    exe = os.path.join(ROOT, "tools", "_build", "e2e_header")
    if not os.path.exists(exe):
        return {"unavailable": "tools/_build/e2e_header not built (__graft_entry__.build())"}
    r = subprocess.run([exe, str(n), str(steps), "2"], capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        return {"unavailable": f"e2e_header failed: {r.stderr[-300:]}"}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    d["value"] = flops_dense(n) / (d["ms_per_step"] * 1e-3) / 1e12
    d["unit"] = "TFLOP/s"
    d["api"] = "randla::preprocess_solve (include/randla_b200/randla.hpp), pageable RealMatrix / std::vector"
    return d


# ---- our arm ---------------------------------------------------------------------
def run_b200(args):
    import torch
    rank, world, local = dist_info()
    if args.dry_run:
        return run_dry(args, rank, world, local)
    if not torch.cuda.is_available():
        print(json.dumps({"error": "no CUDA device"}))
        return 1
    D = Dist(world, local, "nccl")
    torch.cuda.set_device(local)
    import paper_1406_5802_b200 as rl
    from paper_1406_5802_b200 import capi, shard
    L = capi.lib()
    assert L.rl_context_device(None) == local, "the library's default context must follow the rank's device"
    n = args.n
    stream = torch.cuda.current_stream()
    L.rl_context_set_stream(None, ctypes.c_void_p(stream.cuda_stream))

    # inputs (exact reference generator), resident in HBM; 512 MiB each > L2
    A = rl.gen_gaussian(n, n, 1)
    G = rl.gen_gaussian(n, n, 2)
    b = rl.gen_gaussian_vector(n, 3)
    dA, dG, db = torch.from_numpy(A).cuda(), torch.from_numpy(G).cuda(), torch.from_numpy(b).cuda()
    dx = torch.empty_like(db)
    mult = capi.rl_multiplier()
    mult.kind = capi.RL_MULT_GAUSSIAN
    mult.dense = dG.data_ptr()
    info = capi.rl_solve_info()

    def step():
        rc = L.rl_preprocessed_genp_solve(None, capi.RL_DEVICE, n, dA.data_ptr(), db.data_ptr(), None,
                                          ctypes.byref(mult), 0, dx.data_ptr(), None, 0, ctypes.byref(info))
        if rc != 0:
            raise RuntimeError(f"rl_preprocessed_genp_solve failed: {rc} {capi.last_error()}")

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    D.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.2)
    launches0 = L.rl_kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prod_ms = []
    e0.record(stream)
    for _ in range(args.steps):
        step()
        prod_ms.append(info.stage_ms[0])
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    launches = L.rl_kernel_launches() - launches0
    D.barrier()
    clocks = sampler.stop()
    ms = D.max(e0.elapsed_time(e1) / args.steps)
    F = flops_dense(n)
    value = world * F / (ms * 1e-3) / 1e12
    stage = list(info.stage_ms)
    resid = info.residual_history[0]
    growth = info.growth
    x_dev = dx.cpu().numpy()

    # roofline of the dominant kernel: the A*G DMMA GEMM (2 n^3 flops per launch)
    gemm_ms = statistics.mean(prod_ms)
    gemm_tf = 2.0 * n ** 3 / (gemm_ms * 1e-3) / 1e12
    traffic = profiled_traffic("dgemm")
    roofline = {"bound": "tensor", "kernel": "dgemm_kernel (A*G, FP64 DMMA)", "achieved": gemm_tf,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": gemm_tf / FP64_PEAK_TFLOPS, "traffic": traffic,
                "peak_source": "measured on this pool: cuBLAS DGEMM 8192^3 burst (profiles/r01_fp64_peak.txt); "
                               "MEASURED_PEAKS.json carries no FP64 entry",
                "step_frac_of_peak": value / world / FP64_PEAK_TFLOPS,
                "algorithmic_flops_per_launch": 2 * n ** 3}

    e2e = None
    e2e_cpp = None
    if not args.no_e2e:
        e2e = e2e_python(rl, torch, A, b, n, args.e2e_steps, D, world, x_dev)
        if rank == 0 and world == 1:
            e2e_cpp = e2e_cpp_header(n, args.e2e_steps)
        if e2e_cpp is not None:
            e2e["pageable_cpp_header"] = e2e_cpp

    # secondary: BASELINE config 2 (65,536 batched 32x32 systems per GPU), device resident
    secondary = None
    if not args.no_secondary:
        # rank r owns systems [lo, hi) of world * nb (independent
        # systems shard with no data-path collective; weak scaling)
        nb = args.batch
        lo, hi = shard.shard_bounds(world * nb, rank, world)
        ha, hg, hb = shard.shard_inputs(lo, hi)
        ba, bg, bb = (torch.from_numpy(t).cuda() for t in (ha, hg, hb))
        blu, bx = torch.empty_like(ba), torch.empty_like(bb)
        br = torch.empty(nb, dtype=torch.float64, device="cuda")
        bgr = torch.empty_like(br)
        bst = torch.empty(nb, dtype=torch.int32, device="cuda")

        def bstep():
            rc = L.rl_batched_genp_solve_32(None, capi.RL_DEVICE, nb, ba.data_ptr(), bg.data_ptr(), bb.data_ptr(),
                                            blu.data_ptr(), bx.data_ptr(), br.data_ptr(), bgr.data_ptr(),
                                            bst.data_ptr(), None)
            if rc != 0:
                raise RuntimeError(capi.last_error())
        for _ in range(3):
            bstep()
        torch.cuda.synchronize()
        D.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bk = max(args.steps, 10)
        f0.record(stream)
        for _ in range(bk):
            bstep()
        f1.record(stream)
        f1.synchronize()
        bms = D.max(f0.elapsed_time(f1) / bk)
        gbs = nb * BATCH_BYTES_PER_SYSTEM / (bms * 1e-3) / 1e9
        hbm = measured_peaks().get("hbm_gbs", 6534.5)
        summ = shard.reduce_summary(shard.local_summary(br.cpu().numpy(), bgr.cpu().numpy(), bst.cpu().numpy()),
                                    D.dist, device="cuda")
        secondary = {"metric": "batched 32x32 preprocessed GENP solves/s (BASELINE config 2)",
                     "value": world * nb / (bms * 1e-3), "unit": "solves/s", "ms_per_step": bms,
                     "systems_per_gpu": nb, "systems": world * nb, "sharding": "contiguous system blocks per rank",
                     "zero_pivots": summ["zero_pivots"], "max_residual": summ["max_residual"],
                     "max_growth": summ["max_growth"], "mean_residual": summ["mean_residual"],
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                  "traffic": profiled_traffic("batched", nb), "algorithmic_bytes_per_system": BATCH_BYTES_PER_SYSTEM}}
        del ba, bg, bb, blu, bx

    configs = None
    if not args.no_secondary and not args.no_configs and rank == 0:
        del dA, dG
        torch.cuda.empty_cache()
        configs = measure_configs_3_to_5(rl, capi, L, torch, stream, measured_peaks().get("hbm_gbs", 6534.5))

    # CPU baseline: a bounded sample of the same workload on the host cores (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        tf, cinfo = port_sample(n, cores)
        cpu = {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": cinfo["kind"], "sample": cinfo["sample"],
               "seconds": cinfo["seconds"]}

    D.close()
    if rank != 0:
        return 0
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: exact reference RNG, A=gen_gaussian(n,n,1), G=gen_gaussian(n,n,2), b=gen_gaussian_vector(n,3)",
            "config": base_config(n, world),
            "frac_of_fp64_peak": value / world / FP64_PEAK_TFLOPS,
            "stage_ms_last_step": {"product": stage[0], "factor_and_verdict": stage[1], "solve": stage[2],
                                   "call": stage[3]},
            "residual_b": resid, "growth": growth,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": int(launches),
            "secondary": secondary, "configs_3_to_5": configs}
    print(json.dumps(line), flush=True)
    return 0


def run_dry(args, rank, world, local):
    """launcher + collectives without a GPU (gloo): the shape of the N-rank line"""
    D = Dist(world, local, "gloo")
    D.barrier()
    t = D.max(float(rank + 1))
    D.close()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "max_over_ranks_probe": t,
                          "config": base_config(args.n, world)}), flush=True)
    return 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--dry-run", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
