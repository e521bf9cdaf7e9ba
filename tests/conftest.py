import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

# Thread ranks sharing one GPU (ThreadComm peer tests) need eager module loading: under lazy loading
# a kernel's first launch can wait on another rank's spinning peer collective (rs_peer_connect_local
# refuses to connect them otherwise).  Read when CUDA initialises, i.e. after this import.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
# ... and one hardware work queue per stream (the default 8 are shared between streams: a rank's
# kernel queued behind another rank's spinning collective never starts)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


class GoldenCsr:
    """CSR arrays of a golden case in the reference layout."""

    def __init__(self, z, name):
        self.row_ptr = z[f"{name}__row_ptr"]
        self.col_idx = z[f"{name}__col_idx"]
        self.values = z[f"{name}__values"]
        self.nrows = self.ncols = self.n = len(self.row_ptr) - 1


@pytest.fixture(scope="session")
def sweeps_golden():
    with np.load(GOLDEN / "sweeps.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def generators_golden():
    with np.load(GOLDEN / "generators.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def gmres_golden():
    return json.loads((GOLDEN / "gmres.json").read_text())


SWEEP_CASES = ("lap2d_12", "lap3d_8", "lap3d_6x5x4", "ela3d_3", "rand_80", "spd_50", "cd3d_6")


@pytest.fixture(scope="session")
def stationary_golden():
    return json.loads((GOLDEN / "stationary.json").read_text())
