import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_built():
    # oracle (test infrastructure) and the product library; both are in-tree
    # builds that normally already exist (__graft_entry__.build()).
    import oracle
    if oracle.C is None:
        oracle.build()
    import importlib.util
    spec = importlib.util.spec_from_file_location("_rl_build", os.path.join(ROOT, "paper_1406_5802_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()  # incremental: no-op when up to date


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz")))


@pytest.fixture(scope="session")
def orc():
    import importlib
    import oracle
    importlib.reload(oracle) if oracle.C is None else None
    return oracle


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
