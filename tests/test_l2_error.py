"""L2 error of the convergence harness, host side."""

import numpy as np

from paper_2207_03921_b200 import build_ansatz, generate_structured_mesh, perturb
from paper_2207_03921_b200.manufactured import problem_fractional, problem_peridynamic
from paper_2207_03921_b200.solve import interpolate, l2_error


def test_linear_interpolant_is_exact():
    m = perturb(generate_structured_mesh(1.0, 0.25, 8), amplitude=0.2, seed=1)
    for n in (1, 2):
        ans = build_ansatz(m, "cg", n)

        def u(x):
            v = 1.5 + 2.0 * x[..., 0] - 0.5 * x[..., 1]
            return v if n == 1 else np.stack([v, -v], axis=-1)
        c = interpolate(u, m, ans)
        assert l2_error(c, u, m, ans) <= 1e-14


def test_zero_against_one_on_unit_area():
    m = generate_structured_mesh(1.0, 0.0, 6)  # all-domain mesh of [0, 1]^2
    ans = build_ansatz(m)
    e = l2_error(np.zeros(ans.dof_count), lambda x: np.ones(x.shape[:-1]), m, ans)
    assert abs(e - 1.0) <= 1e-14


def test_interpolation_error_rate_two():
    p = problem_fractional()
    errs = []
    for n in (5, 10, 20):
        m = generate_structured_mesh(1.0, 0.0, n)
        ans = build_ansatz(m)
        errs.append(l2_error(interpolate(p.u_exact, m, ans), p.u_exact, m, ans))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(rates - 2.0) <= 0.15), rates


def test_dg_and_vector_interpolants():
    m = generate_structured_mesh(1.0, 0.0, 4)
    p = problem_peridynamic()
    for kind in ("cg", "dg"):
        ans = build_ansatz(m, kind, 2)
        c = interpolate(p.u_exact, m, ans)
        assert c.shape == (ans.dof_count,)
        assert l2_error(c, p.u_exact, m, ans) < 0.05
