"""Pinned L2 errors of the Table 2 study for tests/test_gpu_solve.py.

Runs the study of solve.run_study on the CPU: the oracle's assembly (bit-
identical to the reference, test infrastructure) and load vector, the
Dirichlet split solved with scipy's direct spsolve, and solve.l2_error.
    python tests/golden/make_study.py
"""
import os
import sys

import numpy as np
from scipy.sparse.linalg import spsolve

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import oracle  # noqa: E402
from paper_2207_03921_b200 import (build_adjacency_graph, build_ansatz, fractional_kernel,  # noqa: E402
                                   generate_structured_mesh)
from paper_2207_03921_b200.manufactured import problem_fractional  # noqa: E402
from paper_2207_03921_b200.solve import interpolate, l2_error  # noqa: E402

p, k = problem_fractional(), fractional_kernel(0.5, 0.2)
for n in (5, 10, 20, 40):
    m = generate_structured_mesh(0.5, 0.2, n)
    ans = build_ansatz(m)
    A, _ = oracle.assemble(m, build_adjacency_graph(m), k, ans)
    b = oracle.assemble_load(m, ans, p.f)
    g = interpolate(p.g, m, ans)
    free, cons = np.flatnonzero(ans.free_mask), np.flatnonzero(~ans.free_mask)
    u = g.copy()
    Af = A[free]
    u[free] = spsolve(Af[:, free].tocsc(), b[free] - Af[:, cons] @ g[cons])
    print(n, len(free), repr(l2_error(u, p.u_exact, m, ans)))
