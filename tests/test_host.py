"""CPU tests of the host side: generators, containers, validation, the C ABI surface.

No compute call here touches a GPU; the CUDA parity tests are in test_gpu_*.py.
"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import _native, build, problems

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("name,make", [
    ("laplace2d_5x4", lambda: problems.laplace2d(5, 4)),
    ("laplace3d_4x3x2", lambda: problems.laplace3d(4, 3, 2)),
    ("laplace3d_5", lambda: problems.laplace3d(5)),
    ("elasticity3d_2x3x2", lambda: problems.elasticity3d(2, 3, 2)),
    ("elasticity3d_3", lambda: problems.elasticity3d(3)),
    ("elasticity3d_4_nu0.3", lambda: problems.elasticity3d(4, nu=0.3)),
    ("convdiff3d_5", lambda: problems.convdiff3d(5, (1.0, 0.5, 0.25))),
])
def test_generators_bitwise(name, make, generators_golden):
    a = make()
    assert np.array_equal(a.row_ptr, generators_golden[f"{name}__row_ptr"])
    assert np.array_equal(a.col_idx, generators_golden[f"{name}__col_idx"])
    assert np.array_equal(a.values, generators_golden[f"{name}__values"])


def test_golden_sweep_matrices_match_generators(sweeps_golden):
    for name, a in (("lap2d_12", problems.laplace2d(12)), ("lap3d_8", problems.laplace3d(8)),
                    ("lap3d_6x5x4", problems.laplace3d(6, 5, 4)), ("ela3d_3", problems.elasticity3d(3)),
                    ("cd3d_6", problems.convdiff3d(6, (50.0, 25.0, 10.0)))):
        assert np.array_equal(a.row_ptr, sweeps_golden[f"{name}__row_ptr"]), name
        assert np.array_equal(a.col_idx, sweeps_golden[f"{name}__col_idx"]), name
        assert np.array_equal(a.values, sweeps_golden[f"{name}__values"]), name


def test_random_rhs_host_bitwise(generators_golden):
    for k, want in generators_golden.items():
        if k.startswith("rhs__"):
            _, n, s = k.split("__")
            assert np.array_equal(problems.random_rhs(int(n[1:]), int(s[1:])), want), k
    assert np.array_equal(problems.random_rhs(10, 5), problems.random_rhs(20, 5)[:10])
    assert problems.random_rhs(0).shape == (0,)
    with pytest.raises(ValueError):
        problems.random_rhs(-1)


class TestCsrInvariants:
    """Mirrors test_sparse.py::TestCsrInvariants of the reference."""

    def test_valid(self):
        a = g2.CsrMatrix(2, 2, [0, 2, 3], [0, 1, 1], [1.0, 2.0, 3.0])
        assert a.nnz == 3 and a.precision == "double"

    @pytest.mark.parametrize("args,match", [
        ((2, 2, [1, 2, 3], [0, 1, 1], [1.0, 2.0]), "row_ptr"),
        ((2, 2, [0, 2, 1], [0, 1, 1], [1.0, 2.0, 3.0]), "non-decreasing"),
        ((2, 2, [0, 1, 3], [0, 1], [1.0, 2.0]), "row_ptr"),
        ((2, 2, [0, 1, 2], [0, 2], [1.0, 2.0]), "column index"),
        ((1, 3, [0, 2], [1, 0], [1.0, 2.0]), "strictly increasing"),
        ((1, 3, [0, 2], [1, 1], [1.0, 2.0]), "strictly increasing"),
    ])
    def test_rejected(self, args, match):
        with pytest.raises(ValueError, match=match):
            g2.CsrMatrix(*args)

    def test_dtype(self):
        with pytest.raises(ValueError, match="dtype"):
            g2.CsrMatrix(1, 1, [0, 1], [0], np.array([1], dtype=np.int32))

    def test_from_coo_sums_duplicates(self):
        a = g2.from_coo(2, 2, [0, 0, 1], [1, 1, 0], [1.0, 2.0, 4.0])
        assert a.nnz == 2 and a.to_dense()[0, 1] == 3.0

    def test_immutable(self):
        a = g2.from_dense([[2.0, -1.0], [-1.0, 2.0]])
        with pytest.raises(AttributeError):
            a.nrows = 3

    def test_cast_overflow(self):
        with pytest.raises(OverflowError, match="entry 1"):
            g2.cast_vector(np.array([1.0, 1e39]), "single")
        with pytest.raises(OverflowError, match="matrix value"):
            g2.cast_matrix(g2.from_dense([[1e39]]), "single")
        with pytest.raises(ValueError, match="precision"):
            g2.cast_vector(np.ones(2), "half")


class TestRelaxConfig:
    @pytest.mark.parametrize("kw", [{"n_t": 0}, {"n_k": 0}, {"n_j": -1}, {"omega": 0.0}, {"omega": -0.5},
                                    {"gamma": 0.0}, {"direction": "sideways"}, {"form": "squished"}])
    def test_invalid(self, kw):
        with pytest.raises(ValueError):
            g2.RelaxConfig(**kw)

    def test_partition(self):
        with pytest.raises(ValueError):
            g2.BlockPartition([0, 5, 3])
        with pytest.raises(ValueError):
            g2.BlockPartition([2, 5])
        assert list(g2.BlockPartition.regular(10, 3).offsets) == [0, 3, 7, 10]

    def test_preconditioner_arg_errors(self):
        a = g2.from_dense([[2.0, -1.0], [-1.0, 2.0]])
        with pytest.raises(ValueError, match="kind"):
            g2.Preconditioner(a, "ilu")
        with pytest.raises(ValueError, match="precision"):
            g2.Preconditioner(a, "jr", precision="half")


def _header_symbols():
    txt = (ROOT / "include" / "gs2b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|int64_t|double|const char \*)\s*(rs_\w+)\(", txt, re.M)))


def test_library_builds_and_exports_every_header_symbol():
    lib_path = build.build()
    lib = ctypes.CDLL(str(lib_path))
    syms = _header_symbols()
    assert len(syms) >= 28
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.exported_symbols())
    assert lib.rs_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(build.build())], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_import_in_product():
    pkg = ROOT / "paper_2104_01196_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        txt = f.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
        assert "liboracle" not in txt and "orc_" not in txt, f


def test_host_givens_is_the_numpy_arithmetic():
    """rs_host_givens (the GMRES Givens step in the library's host code) is bitwise the numpy loop it
    replaces (krylov.py:224-234 arithmetic: separately rounded products and sums, libm hypot)."""
    from paper_2104_01196_b200 import krylov

    rng = np.random.default_rng(3)
    for _ in range(300):
        m = int(rng.integers(1, 70))
        j = int(rng.integers(0, m))
        h = rng.standard_normal((m + 1, m)) * 10.0 ** rng.integers(-8, 8)
        cs, sn, g = rng.standard_normal(m), rng.standard_normal(m), rng.standard_normal(m + 1)
        hf = np.zeros((m + 1, 2 * m))[:, ::2]  # a strided (non-contiguous) copy takes the numpy loop
        hf[...] = h
        cs2, sn2, g2 = cs.copy(), sn.copy(), g.copy()
        r1 = krylov._givens_step(h, cs, sn, g, j)      # library host code (C-contiguous h)
        r2 = krylov._givens_step(hf, cs2, sn2, g2, j)  # numpy loop (the specification)
        assert r1 == r2
        assert np.array_equal(h, hf) and np.array_equal(cs, cs2) and np.array_equal(sn, sn2)
        assert np.array_equal(g, g2)
