"""Dirichlet split + device CG against scipy's direct
solve of the same split system."""

import numpy as np
import pytest
from scipy.sparse.linalg import spsolve

from golden_io import Case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", ["cfg1_approxcaps", "frac_s04_approx_pert", "peri_nocaps_avoid"])
def test_dirichlet_cg_matches_direct_solve(name):
    from paper_2207_03921_b200 import assemble_load, bfs_assemble
    from paper_2207_03921_b200.solve import solve_dirichlet
    c = Case(name)
    sysm = bfs_assemble(*c.args(), rows=c.rows)
    b = assemble_load(c.mesh, c.ansatz, c.f, c.quad)
    u, info = solve_dirichlet(sysm, b, rtol=1e-13)
    a_ff, _ = sysm.split()
    free = np.flatnonzero(sysm.free_mask)
    ref = spsolve(a_ff.tocsc(), b[free])
    assert info["relres"] <= 1e-13
    assert np.linalg.norm(u[free] - ref) <= 1e-9 * np.linalg.norm(ref)
    assert np.all(u[~sysm.free_mask] == 0.0)


def test_cg_deterministic_and_dirichlet_data():
    from paper_2207_03921_b200 import assemble_load, bfs_assemble
    from paper_2207_03921_b200.solve import solve_dirichlet
    c = Case("cfg1_nocaps")
    sysm = bfs_assemble(*c.args(), rows=c.rows)
    b = assemble_load(c.mesh, c.ansatz, c.f, c.quad)
    g = np.where(sysm.free_mask, 0.0, 0.25)
    u1, i1 = solve_dirichlet(sysm, b, g=g, rtol=1e-12)
    u2, i2 = solve_dirichlet(sysm, b, g=g, rtol=1e-12)
    assert np.array_equal(u1, u2) and i1 == i2
    assert np.all(u1[~sysm.free_mask] == 0.25)
    r = sysm.matrix @ u1 - b
    assert np.linalg.norm(r[sysm.free_mask]) <= 1e-10 * np.linalg.norm(b[sysm.free_mask])
