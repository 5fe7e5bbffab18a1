"""N>1 host logic of the batched path on CPU: world_size-2
gloo processes each take their shard of BASELINE config 2's systems
(shard.shard_bounds + the reference's per-trial seed derivation), solve it
with the CPU oracle as a stand-in for the per-GPU kernel, and all-reduce the
summary; the result must equal one process solving every system."""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1406_5802_b200 import shard

TOTAL = 96


def test_shard_bounds_cover_exactly():
    for total in (0, 1, 7, 96, 65536, 65537):
        for world in (1, 2, 3, 8):
            spans = [shard.shard_bounds(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.shard_bounds(10, 2, 2)


def test_batch_seeds_match_oracle_inputs(orc):
    import paper_1406_5802_b200 as rl
    lo, hi = 5, 9
    seeds = shard.batch_seeds(lo, hi)
    ref = orc.C.batched_config2(hi - lo, base=7, i0=lo)
    np.testing.assert_array_equal(rl.gen_gaussian_batch(hi - lo, 32, 32, seeds[:, 0]), ref["a"])
    np.testing.assert_array_equal(rl.gen_gaussian_batch(hi - lo, 32, 1, seeds[:, 1]).reshape(-1, 32), ref["b"])
    np.testing.assert_array_equal(rl.gen_gaussian_batch(hi - lo, 32, 32, seeds[:, 2]), ref["g"])


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard.shard_bounds(TOTAL, rank, world)
    r = oracle.C.batched_config2(hi - lo, base=7, i0=lo, want_inputs=False)
    local = shard.local_summary(r["resid"], r["growth"], r["status"])
    total = shard.reduce_summary(local, dist, device="cpu")
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"lo": lo, "hi": hi, "local": local, "total": total, "x": r["x"].tolist()}, f)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_shards_equal_single_process(orc, tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    outs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    full = orc.C.batched_config2(TOTAL, base=7, i0=0, want_inputs=False)
    want = shard.reduce_summary(shard.local_summary(full["resid"], full["growth"], full["status"]))
    # both ranks hold the same reduced summary, equal to the one-process run
    for o in outs:
        t = o["total"]
        assert t["max_growth"] == want["max_growth"]
        assert t["max_residual"] == want["max_residual"]
        assert t["zero_pivots"] == want["zero_pivots"] and t["counted"] == want["counted"] == TOTAL
        assert abs(t["sum_residual"] - want["sum_residual"]) <= 1e-12 * want["sum_residual"]
    # and the shards are exactly the single-process systems
    x = np.concatenate([np.array(o["x"]) for o in outs])
    np.testing.assert_array_equal(x, full["x"])


def _fake_device_entry(orc):
    """rl_batched_genp_solve_32 replaced by a host stand-in that reads and
    writes exactly the pointers and sizes the library call passes (this CPU
    box has no device); everything above it is the product's plumbing."""
    import ctypes

    def fake(ctx, mem, batch, a, g, b, lu, x, resid, growth, status, summary):
        assert mem == 0  # host arrays in, as a numpy caller passes them
        dp = ctypes.POINTER(ctypes.c_double)
        view = lambda p, n: np.ctypeslib.as_array(ctypes.cast(p, dp), shape=(n,))  # noqa: E731
        A = view(a, batch * 1024).reshape(batch, 32, 32)
        G = view(g, batch * 1024).reshape(batch, 32, 32)
        B = view(b, batch * 32).reshape(batch, 32)
        X = view(x, batch * 32).reshape(batch, 32)
        R, GR = view(resid, batch), view(growth, batch)
        ST = np.ctypeslib.as_array(ctypes.cast(status, ctypes.POINTER(ctypes.c_int32)), shape=(batch,))
        for i in range(batch):
            o = orc.C.preprocess_solve(A[i], B[i], 1, G[i], refine=0, want_lu=True)
            X[i] = o["x"]
            R[i] = o["history"][0]
            ST[i] = o["zero_step"]
            GR[i] = np.abs(np.triu(o["lu"])).max() / np.abs(o["product"]).max()
        return 0
    return fake


def _worker_plumbing(rank, world, port, out_dir):
    import torch.distributed as dist
    import oracle
    from paper_1406_5802_b200 import capi
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = capi.lib()

    class Patched:  # the library with its device entry point swapped for the host stand-in
        def __getattr__(self, name):
            return getattr(lib, name)
    patched = Patched()
    patched.rl_batched_genp_solve_32 = _fake_device_entry(oracle)
    capi._lib = patched
    lo, hi, out, total = shard.run_batched_shard(TOTAL, rank, world, dist, device="cpu")
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"lo": lo, "hi": hi, "total": total, "x": out.x.tolist()}, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_library_plumbing_equals_single_process(orc, tmp_path):
    """world_size-2 gloo ranks run shard.run_batched_shard -> the library's
    randla.batched_preprocess_solve_32 -> the C entry point (host stand-in):
    the concatenated solutions and the reduced summary equal one process
    solving every system."""
    world = 2
    mp.spawn(_worker_plumbing, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    outs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    assert [(o["lo"], o["hi"]) for o in outs] == [shard.shard_bounds(TOTAL, r, world) for r in range(world)]
    full = orc.C.batched_config2(TOTAL, base=7, i0=0, want_inputs=False)
    np.testing.assert_array_equal(np.concatenate([np.array(o["x"]) for o in outs]), full["x"])
    want = shard.reduce_summary(shard.local_summary(full["resid"], full["growth"], full["status"]))
    for o in outs:
        assert o["total"]["counted"] == TOTAL and o["total"]["zero_pivots"] == want["zero_pivots"]
        assert o["total"]["max_residual"] == want["max_residual"]
