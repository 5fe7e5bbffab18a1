#!/usr/bin/env python
"""Benchmark driver (one JSON line on rank 0).

Workload (BASELINE.json metric "preprocessed-GENP FP64 TFLOP/s at n=8192, % of
FP64 peak; batched solves/s"): one step = one Gaussian-preprocessed GENP
solve at n=8192 — preprocess_solve(A, b, none, {Gaussian, G}, 0)
(preprocess.hpp:156-180): product A*G, blocked GENP with the pivot verdict,
chain solve x = G (LU)^-1 b — with A (seed 1), G (seed 2), b (seed 3) resident
in HBM. value = F(n) / step time in TFLOP/s, F(n) = (2n^3 - n^2) +
sum_{m<n} m(1+2m) + 2n^2 + (2n^2 - n). The batched-32
figure (BASELINE config 2, 65,536 systems) rides along under "secondary".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: the reference headers compiled with our Eigen shim; the plain-C
port when _ref is absent) on all host cores, running preprocess_solve trials
concurrently on the reference's parallel_for_index pool, on a bounded sample
(n=2048 per trial) in the same metric/unit.

Multi-GPU (torchrun): every rank solves its own n=8192 system (the dense
path does not shard: replicas only); value = all ranks' flops /
max-over-ranks step time.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "preprocessed-GENP FP64 TFLOP/s at n=8192, % of FP64 peak; batched solves/s"
FP64_PEAK_TFLOPS = 35.46   # cuBLAS DGEMM 8192^3 measured on this pool's B200 (profiles/r01_fp64_peak.txt)
FP64_DMMA_PEAK = 37.06     # DMMA issue-rate microbenchmark (tools/fp64_peak.cu)
BATCH_BYTES_PER_SYSTEM = 25104


def flops_dense(n):
    """F(n) of SURVEY §8(d)."""
    s = n * (n - 1) // 2 + 2 * ((n - 1) * n * (2 * n - 1) // 6)
    return (2 * n ** 3 - n ** 2) + s + 2 * n ** 2 + (2 * n ** 2 - n)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


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
    def __init__(self, world, local):
        import torch
        self.torch = torch
        self.world = world
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            self.dist = dist
        else:
            self.dist = None

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, v):
        if not self.dist:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# ---- the reference arm ---------------------------------------------------------
def reference_sample(n_s, trials, steps, warmup):
    """Time the reference CPU path: `trials` concurrent preprocess_solve calls
    (n_s x n_s Gaussian A, Gaussian multiplier) per step. Returns (TF/s, info)."""
    import oracle
    seeds = np.array([oracle.C.derive_seed(1000 + t, 2, 0) for t in range(trials)], dtype=np.uint64)
    a_all = np.stack([oracle.C.gen_gaussian(n_s, n_s, oracle.C.derive_seed(1000 + t, 1, 0)) for t in range(trials)])
    b_all = np.stack([oracle.C.gen_gaussian_vector(n_s, oracle.C.derive_seed(1000 + t, 3, 0)) for t in range(trials)])
    if oracle.REF is not None:
        kind = "reference"

        def step():
            res, nf = oracle.REF.parallel_dense_trials(a_all, b_all, seeds)
            return res
    else:
        kind = "port"

        def step():
            out = [None] * trials

            def work(t):
                g = oracle.C.gen_gaussian(n_s, n_s, int(seeds[t]))
                out[t] = oracle.C.preprocess_solve(a_all[t], b_all[t], 1, g)["history"][0]
            th = [threading.Thread(target=work, args=(t,)) for t in range(trials)]
            for x in th:
                x.start()
            for x in th:
                x.join()
            return np.array(out)
    for _ in range(warmup):
        step()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        res = step()
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    tf = trials * flops_dense(n_s) / t / 1e12
    return tf, {"kind": kind, "cores": trials, "seconds_per_step": t, "median_residual": float(np.nanmedian(res)),
                "sample": f"{trials} concurrent preprocess_solve trials, n={n_s} (Gaussian A, Gaussian multiplier, "
                          f"refine 0) per step on the reference's parallel_for_index pool; metric scaled by F(n)"}


def run_reference(args):
    rank, world, local = dist_info()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    tf, info = reference_sample(args.ref_n, cores, max(1, args.steps), max(0, args.warmup))
    line = {"impl": "reference", "metric": METRIC, "value": tf, "unit": "TFLOP/s", "n_gpus": 0, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": info["seconds_per_step"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded reference RNG)",
            "config": {"workload": f"reference CPU preprocess_solve, bounded sample n={args.ref_n} x {cores} trials",
                       "n_sample": args.ref_n, "trials_per_step": cores},
            "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": info["kind"],
                             "sample": info["sample"]},
            "e2e": {"value": tf, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---- BASELINE configs 3-5 (device resident, one timed call each) ---------------
def measure_configs_3_to_5(rl, capi, L, torch, stream, hbm):
    """Config 3: circulant-preprocessed GENP at n=8192 (FFT product + blocked
    GENP + FFT chain solve); config 4: range finder m=n=8192, r=64, Gaussian H;
    config 5: m=32768, n=16384, r=256, Toeplitz H by FFT. Inputs follow
    BASELINE.json (Haar factors from QR of seeded N(0,1) matrices); E and the
    large Gaussian factors are drawn on the device with torch's seeded
    generator (untimed input construction)."""
    out = {}

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

    # ---- config 3
    n = 8192
    gu = torch.from_numpy(rl.gen_gaussian(n, n, 11)).cuda()
    u, _ = torch.linalg.qr(gu)
    del gu
    gv = torch.from_numpy(rl.gen_gaussian(n, n, 12)).cuda()
    v, _ = torch.linalg.qr(gv)
    del gv
    a = (u * torch.logspace(0, -4, n, dtype=torch.float64, device="cuda")) @ v.T
    del u, v
    b = torch.from_numpy(rl.gen_gaussian_vector(n, 14)).cuda()
    c = torch.from_numpy(rl.gen_gaussian_vector(n, 13)).cuda()
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
        rc = L.rl_preprocessed_genp_solve(None, capi.RL_DEVICE, n, a.data_ptr(), b.data_ptr(), ctypes.byref(m3), 0,
                                          x.data_ptr(), None, 0, ctypes.byref(info))
        if rc != 0:
            raise RuntimeError(capi.last_error())
    ms3 = ev_time(solve3, 2)
    lu_flops = sum_lu_flops(n)
    fft_bytes = 2 * 8 * n * n
    out["config3"] = {
        "workload": "circulant-preprocessed GENP, n=8192, kappa=1e4 (Haar U/V seeds 11/12), Gaussian circulant seed 13",
        "ms_per_call": ms3, "stage_ms": list(info.stage_ms), "residual_b": info.residual_history[0],
        "growth": info.growth,
        "fft_product": {"ms": fft_ms, "roofline": {"bound": "hbm", "achieved": fft_bytes / (fft_ms * 1e-3) / 1e9,
                                                    "peak": hbm, "unit": "GB/s",
                                                    "frac": fft_bytes / (fft_ms * 1e-3) / 1e9 / hbm,
                                                    "algorithmic_bytes": fft_bytes}},
        "lu_tflops": lu_flops / (info.stage_ms[1] * 1e-3) / 1e12}
    del a, b, c, x

    # ---- config 4
    m = n = 8192
    r = 64
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    ur, _ = torch.linalg.qr(torch.randn(m, r, dtype=torch.float64, device="cuda", generator=g))
    vr, _ = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g))
    sig = torch.logspace(0, -2, r, dtype=torch.float64, device="cuda")
    a = (ur * sig) @ vr.T + 1e-10 * torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    out["config4"] = run_range_find(L, capi, a, r, capi.RL_MULT_GAUSSIAN, 41, ev_time, 3 * 2 * m * n * r,
                                    "range finder m=n=8192, r=64, Gaussian H (seed 41); sigma 1..1e-2, E ~ N(0,1e-20)")
    del a, ur, vr

    # ---- config 5
    m, n, r = 32768, 16384, 256
    g.manual_seed(5)
    ur, _ = torch.linalg.qr(torch.randn(m, r, dtype=torch.float64, device="cuda", generator=g))
    vr, _ = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g))
    sig = torch.logspace(0, -3, r, dtype=torch.float64, device="cuda")
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g).mul_(1e-12)
    a.addmm_(ur * sig, vr.T)
    del ur, vr
    res5 = run_range_find(L, capi, a, r, capi.RL_MULT_GAUSSIAN_CIRCULANT, 21, ev_time, 2 * 2 * m * n * r,
                          "range finder m=32768, n=16384, r=256, Toeplitz H (Gaussian circulant seed 21); "
                          "sigma 1..1e-3, E ~ N(0,1e-24)")
    # the Toeplitz sketch alone (HBM bound: read A, write Y)
    cc = torch.from_numpy(rl.gen_gaussian_vector(n, 21)).cuda()
    y = torch.empty(m, r, dtype=torch.float64, device="cuda")
    sk_ms = ev_time(lambda: L.rl_toeplitz_right_multiply(None, capi.RL_DEVICE, m, n, a.data_ptr(), n, cc.data_ptr(), r,
                                                         y.data_ptr()), 1)
    sk_bytes = 8 * m * n + 8 * m * r
    res5["toeplitz_sketch"] = {"ms": sk_ms, "roofline": {"bound": "hbm", "achieved": sk_bytes / (sk_ms * 1e-3) / 1e9,
                                                         "peak": hbm, "unit": "GB/s",
                                                         "frac": sk_bytes / (sk_ms * 1e-3) / 1e9 / hbm,
                                                         "algorithmic_bytes": sk_bytes}}
    out["config5"] = res5
    del a, y
    torch.cuda.empty_cache()
    return out


def sum_lu_flops(n):
    return n * (n - 1) // 2 + 2 * ((n - 1) * n * (2 * n - 1) // 6)


def run_range_find(L, capi, a, r, kind, seed, ev_time, gemm_flops, workload):
    m, n = a.shape
    q = a.new_empty(m, r)
    mlt = capi.rl_multiplier()
    mlt.kind = kind
    mlt.seed = seed
    info = capi.rl_lowrank_info()

    def call():
        rc = L.rl_range_find_residual(None, capi.RL_DEVICE, m, n, a.data_ptr(), r, ctypes.byref(mlt), q.data_ptr(),
                                      ctypes.byref(info))
        if rc != 0:
            raise RuntimeError(capi.last_error())
    ms = ev_time(call, 1)
    return {"workload": workload, "ms_per_call": ms, "residual_frobenius": info.residual_frobenius,
            "residual_spectral": info.residual_spectral, "power_iterations": info.power_iterations,
            "product_tflops_equiv": gemm_flops / (ms * 1e-3) / 1e12,
            "note": "call = sketch + CholeskyQR2 + Q^T A + residual ||.||_F + power-iteration ||.||_2"}


# ---- our arm ---------------------------------------------------------------------
def run_b200(args):
    import torch
    rank, world, local = dist_info()
    if not torch.cuda.is_available():
        print(json.dumps({"error": "no CUDA device"}))
        return 1
    D = Dist(world, local)
    torch.cuda.set_device(local)
    import paper_1406_5802_b200 as rl
    from paper_1406_5802_b200 import capi
    L = capi.lib()
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
        rc = L.rl_preprocessed_genp_solve(None, capi.RL_DEVICE, n, dA.data_ptr(), db.data_ptr(), ctypes.byref(mult), 0,
                                          dx.data_ptr(), None, 0, ctypes.byref(info))
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

    # roofline of the dominant kernel: the A*G DMMA GEMM (2 n^3 flops per launch)
    gemm_ms = statistics.mean(prod_ms)
    gemm_tf = 2.0 * n ** 3 / (gemm_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r01_dgemm_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": "dgemm_kernel (A*G, FP64 DMMA)", "achieved": gemm_tf,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": gemm_tf / FP64_PEAK_TFLOPS, "traffic": traffic,
                "peak_source": "measured on this pool: cuBLAS DGEMM 8192^3 burst (profiles/r01_fp64_peak.txt); "
                               "MEASURED_PEAKS.json carries no FP64 entry",
                "step_frac_of_peak": value / world / FP64_PEAK_TFLOPS,
                "algorithmic_flops_per_launch": 2 * n ** 3}

    # end to end through the public API with host buffers: pinned A, b in,
    # the multiplier generated from its seed inside the call (as the
    # reference's preprocess_solve does), x out
    e2e = None
    if not args.no_e2e:
        hA = torch.from_numpy(A).pin_memory()
        hb = torch.from_numpy(b).pin_memory()
        hx = torch.empty(n, dtype=torch.float64).pin_memory()
        m2 = capi.rl_multiplier()
        m2.kind = capi.RL_MULT_GAUSSIAN
        m2.seed = 2
        info2 = capi.rl_solve_info()

        def e2e_step():
            rc = L.rl_preprocessed_genp_solve(None, capi.RL_HOST, n, hA.data_ptr(), hb.data_ptr(), ctypes.byref(m2), 0,
                                              hx.data_ptr(), None, 0, ctypes.byref(info2))
            if rc != 0:
                raise RuntimeError(capi.last_error())
        e2e_step()
        D.barrier()
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - t0)
        t = D.max(statistics.mean(ts))
        same = bool(np.array_equal(hx.numpy(), dx.cpu().numpy()))
        e2e = {"value": world * F / t / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 8 * n * n + 8 * n,
               "d2h_bytes_per_step": 8 * n, "ms_per_step": t * 1e3, "steps": args.e2e_steps,
               "includes": "H2D of A (4 row blocks on a side stream, overlapped with the product) and b from "
                           "pinned memory, exact generation of G from seed 2 on the device (the ~6% of log "
                           "evaluations glibc must decide finished on the host), product, GENP, verdict, solve, "
                           "D2H of x",
               "matches_device_resident_x": same}

    # secondary: BASELINE config 2 (65,536 batched 32x32 systems), device resident
    secondary = None
    if not args.no_secondary:
        # rank r owns systems [lo, hi) of world * nb (independent
        # systems shard with no data-path collective; weak scaling)
        from paper_1406_5802_b200 import shard
        nb = args.batch
        lo, hi = shard.shard_bounds(world * nb, rank, world)
        seeds = shard.batch_seeds(lo, hi)
        ba = torch.from_numpy(rl.gen_gaussian_batch(nb, 32, 32, seeds[:, 0])).cuda()
        bb = torch.from_numpy(rl.gen_gaussian_batch(nb, 32, 1, seeds[:, 1]).reshape(nb, 32)).cuda()
        bg = torch.from_numpy(rl.gen_gaussian_batch(nb, 32, 32, seeds[:, 2])).cuda()
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
                                  "traffic": None, "algorithmic_bytes_per_system": BATCH_BYTES_PER_SYSTEM}}

    configs = None
    if not args.no_secondary and not args.no_configs:
        configs = measure_configs_3_to_5(rl, capi, L, torch, stream, measured_peaks().get("hbm_gbs", 6534.5))

    # CPU baseline: the reference's CPU path on the host cores (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        tf, cinfo = reference_sample(args.ref_n, cores, 1, 0)
        cpu = {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": cinfo["kind"], "sample": cinfo["sample"]}

    D.close()
    if rank != 0:
        return 0
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: exact reference RNG, A=gen_gaussian(n,n,1), G=gen_gaussian(n,n,2), b=gen_gaussian_vector(n,3)",
            "config": {"workload": f"Gaussian-preprocessed GENP solve, n={n} (BASELINE headline; config 1 recipe at "
                                   f"n={n})", "n": n, "refine_steps": 0, "multiplier": "gaussian",
                       "l2": "inputs 1 GiB per step > 126 MB L2 (no flush needed)",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "frac_of_fp64_peak": value / world / FP64_PEAK_TFLOPS,
            "stage_ms_last_step": {"product": stage[0], "factor_and_verdict": stage[1], "solve": stage[2],
                                   "call": stage[3]},
            "residual_b": resid, "growth": growth,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": int(launches),
            "secondary": secondary, "configs_3_to_5": configs}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--ref-n", type=int, default=2048)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
