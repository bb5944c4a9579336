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


def test_table2_fractional_convergence_study():
    """SURVEY 8f row 1 / SPEC.md:459-499: the paper's Table 2 study (fractional
    CG, s = 0.5, delta = 0.2, nocaps, Omega = (0, 0.5)^2, n_div 5..40, free
    dofs 16 / 81 / 361 / 1521 as in the table): assembly, load and Dirichlet
    solve on the GPU, L2 error of the manufactured solution over Omega~.

    * rates within 0.3 of Table 2's {2.13, 2.01, 2.01};
    * errors equal (1e-6 relative: CG vs a direct solve) to the same study
      run with the CPU oracle + scipy spsolve (pinned values below).  The
      paper does not define its error norm; ours (the
      7-point rule on |u_h - u|^2 over Omega~) is a constant factor ~4 above
      the tabulated values at every level, with the same rates.
    """
    from paper_2207_03921_b200 import fractional_kernel
    from paper_2207_03921_b200.manufactured import problem_fractional
    from paper_2207_03921_b200.solve import run_study
    rows = run_study(lambda: fractional_kernel(0.5, 0.2), problem_fractional(), [5, 10, 20, 40])
    for r in rows:
        assert r["cg_relres"] <= 1e-10
    assert [r["dof"] for r in rows] == [16, 81, 361, 1521]
    errs = [r["l2_error"] for r in rows]
    rates = [r["rate"] for r in rows[1:]]
    for got, want in zip(rates, (2.13, 2.01, 2.01)):
        assert abs(got - want) <= 0.3, (rates, errs)
    oracle_errs = (0.002723214856838669, 0.0006639707327425461, 0.00016612007113837868, 4.1585564860848426e-05)
    for got, want in zip(errs, oracle_errs):
        assert abs(got - want) <= 1e-6 * want, (errs, oracle_errs)
