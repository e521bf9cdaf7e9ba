"""The window-pipelined one-launch GS2 sweep (relax.cu k_gs2_pipe) against the multi-pass sweep,
and the multi-pass sweep with its layout / prefetch switches off (variable-width SELL slices, no
software L2 prefetch, one-row fp32 kernels, scalar scale pass) against the default.

Both paths keep the reference's operation forms, so every iterate must be bitwise equal:
GS2 n_j 1/2/3/5, forward / backward / symmetric, non-compact / compact, omega / gamma != 1,
n_t = 2 (consecutive launches), fp64 and fp32, and the zero-start preconditioner (fp64,
fp32, fp32-inside-fp64) on Laplace, convection-diffusion, elasticity and a structurally
non-symmetric banded matrix.  Small windows (RS_PIPE_WS=5: W = the matrix bandwidth rounded
up to a power of two, 8-70 windows) exercise the cross-window dependencies and ring reuse;
the default windows (2^17 rows) give one window per matrix here.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

HERE = Path(__file__).resolve().parent


def _run(tmp_path, tag, **env):
    out = tmp_path / f"{tag}.npz"
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, str(HERE / "pipe_worker.py"), str(out)], env=e, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "PIPE_WORKER_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
    return dict(np.load(out))


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("pipe")
    return {
        "multipass": _run(tmp, "multipass", RS_PIPE="0"),
        "pipe_small": _run(tmp, "pipe_small", RS_PIPE="1", RS_PIPE_WS="5"),
        "pipe_default": _run(tmp, "pipe_default", RS_PIPE="1"),
        # layout / prefetch switches of the default path: variable-width slices (loaded bounds),
        # no software L2 prefetch, one-row fp32 preconditioner kernels
        "varwidth_nopf": _run(tmp, "varwidth_nopf", RS_PIPE="0", RS_SELL_UNIFORM="0", RS_PF_DIST="0",
                              RS_F32_NR="1", RS_SCALE_X2="0"),
    }


@pytest.mark.parametrize("variant", ["pipe_small", "pipe_default", "varwidth_nopf"])
def test_pipe_bitwise_equals_multipass(runs, variant):
    ref, got = runs["multipass"], runs[variant]
    keys = [k for k in ref if not k.startswith("launches:")]
    assert len(keys) > 500 and set(keys) <= set(got)
    bad = [k for k in keys if not np.array_equal(ref[k], got[k])]
    assert not bad, f"{len(bad)} iterates differ, e.g. {bad[:5]}"


def test_pipe_is_one_launch_per_half_sweep(runs):
    # the pipelined path must actually run: a non-compact forward GS2(2,1,n_j) sweep is
    # 2 x (1 + n_j) launches multi-pass, 2 pipelined
    ref, got = runs["multipass"], runs["pipe_small"]
    key = "launches:f64/lap3d_20/sweep/3/forward/non_compact/1.0/1.0"
    assert int(ref[key]) == 8
    assert int(got[key]) <= 4  # + the one-time bandwidth probe (2 launches)
