"""Host logic of the trial engine (paper_1406_5802_b200.testbed): statistics
and per-trial seed derivation as in the reference's testbed
(stats.hpp:19-34, experiment.hpp:30-69), checked against the CPU oracle."""
import math

import numpy as np
import pytest

from paper_1406_5802_b200 import randla as rl
from paper_1406_5802_b200 import testbed


def test_summarize_matches_reference_formula():
    v = [3.0, 1.0, 4.0, 1.0, 5.0, 9.0, 2.0, 6.0]
    s = testbed.summarize(v)
    assert (s.min, s.max) == (1.0, 9.0)
    assert s.mean == sum(v) / len(v)
    assert s.std == math.sqrt(sum((x - s.mean) ** 2 for x in v) / len(v))  # population std
    with pytest.raises(ValueError):
        testbed.summarize([])


def test_trial_seeds_follow_the_reference_derivation(orc):
    seen = {}

    def trial(ts, t):
        seen[t] = ts  # trials may run concurrently (parallel_for_index): key by index
        if t == 3:
            raise rl.ZeroPivotError(1)
        return [float(t), float(ts % 7)]

    rep = testbed.run_experiment("table3/n=64", 6, 42, ["a", "b"], trial, "gaussian", 1, 64)
    key = orc.C.hash_label(b"table3/n=64")
    assert [seen[t] for t in range(6)] == [orc.C.derive_seed(42, key, t) for t in range(6)]
    assert rep.failures == 1 and rep.trials == 6
    assert rep.column("a").values == [0.0, 1.0, 2.0, 4.0, 5.0]
    assert rep.column("a").stats.max == 5.0
    with pytest.raises(rl.DimensionError):
        testbed.run_experiment("x", 0, 1, ["a"], trial)
