"""Pin the CPU oracle (oracle/nlfem_oracle.c) against fixtures the
reference itself produced (tests/golden/make_golden.py): the CSR must be
identical bit for bit -- pattern AND values -- and the load vector within
1e-14 (einsum order differs)."""

import numpy as np
import pytest

from golden_io import Case, names
from oracle import oracle


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


@pytest.mark.parametrize("name", names())
def test_oracle_matches_reference_bitwise(name):
    c = Case(name)
    mat, r = oracle.assemble(*c.args(), rows=c.rows, nthreads=4)
    assert r["err"] == 0
    ref = c.matrix
    assert np.array_equal(mat.indptr, ref.indptr)
    assert np.array_equal(mat.indices, ref.indices)
    assert np.array_equal(mat.data, ref.data), np.abs(mat.data - ref.data).max()


@pytest.mark.parametrize("name", names())
def test_oracle_load_matches_reference(name):
    c = Case(name)
    b = oracle.assemble_load(c.mesh, c.ansatz, c.f, c.quad)
    assert np.linalg.norm(b - c.b) <= 1e-14 * max(np.linalg.norm(c.b), 1e-300)


@pytest.mark.parametrize("name", ["cfg1_nocaps", "frac_s04_approx_pert", "lshape16_const"])
def test_bfs_equals_brute(name):
    c = Case(name)
    a, _ = oracle.assemble(*c.args(), rows=c.rows, traversal="bfs")
    b, _ = oracle.assemble(*c.args(), rows=c.rows, traversal="brute")
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data, b.data)


def test_thread_count_invariance():
    c = Case("frac_s04_approx_pert")
    a, _ = oracle.assemble(*c.args(), nthreads=1)
    b, _ = oracle.assemble(*c.args(), nthreads=7)
    assert np.array_equal(a.data, b.data) and np.array_equal(a.indices, b.indices)


def test_survey_golden_numbers():
    # cfg1 nocaps nnz 57,297, |A|_F = 16.146618353794768, max|A| = 0.5062411566446074
    c = Case("cfg1_nocaps")
    mat, _ = oracle.assemble(*c.args())
    assert mat.nnz == 57297
    assert abs(np.linalg.norm(mat.data) - 16.146618353794768) <= 1e-13
    assert abs(np.abs(mat.data).max() - 0.5062411566446074) <= 1e-15
