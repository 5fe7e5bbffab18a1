"""Run one of the paper's preprocessed-GENP presets on the GPU and print its
report table and the reference's checks (testbed/presets.hpp).
usage: python tools/run_preset.py table3 [seed] [trials] [--full]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1406_5802_b200 import testbed  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "table3"
args = [a for a in sys.argv[2:] if not a.startswith("--")]
seed = int(args[0]) if args else 1
trials = int(args[1]) if len(args) > 1 else 100
t0 = time.time()
reports, checks = testbed.run_preset(name, seed, trials, "--full" in sys.argv)
print(f"{name}: seed {seed}, {trials} trials per dimension, {time.time() - t0:.1f} s")
for r in reports:
    cols = "  ".join(f"{c.name}: mean {c.stats.mean:.3e} max {c.stats.max:.3e}" for c in r.columns)
    print(f"  n={r.dimension:5d}  failures {r.failures:3d}  {cols}")
for c in checks:
    print(f"  [{'PASS' if c.passed else 'FAIL'}] {c.description}")
