"""bench.py's multi-GPU plumbing on CPU: --gpus 2 relaunches itself under
torch.distributed.run (one process per device) and, with --dry-run, runs the
barrier / max-over-ranks collectives over gloo and prints n_gpus = 2."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_dry_run_prints_n_gpus_2():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["max_over_ranks_probe"] == 2.0
    assert lines[0]["config"]["parallelism"] == "replicas x2"
