"""Manufactured problems of the convergence studies.

Restates ``/root/reference/pkg/src/nlfem/kernels.py:121-188``
(``ManufacturedProblem``, ``problem_fractional``, ``problem_peridynamic``,
``problem_infinity``): exact solution, forcing term and Dirichlet data
g = u.  These are host callables -- they feed ``assemble_load`` (which
evaluates f once on the stacked quadrature points) and the L2 error.
"""

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ManufacturedProblem:
    """Exact solution, forcing term, and volume constraint data g = u."""

    n: int
    u_exact: callable
    f: callable
    g: callable


def problem_fractional():
    """u = x1^2 x2 + x2^2, f = -2 (x2 + 1) (the scaled operator reproduces the
    Laplacian on cubic polynomials)."""

    def u(x):
        x = np.asarray(x, dtype=float)
        return x[..., 0] ** 2 * x[..., 1] + x[..., 1] ** 2

    def f(x):
        x = np.asarray(x, dtype=float)
        return -2.0 * (x[..., 1] + 1.0)

    return ManufacturedProblem(n=1, u_exact=u, f=f, g=u)


def problem_peridynamic():
    """u = (x2^2, x1^2 x2), f = -(pi/2) (1 + 2 x1, x2) (local elastic limit
    of the 3/delta^3-scaled operator)."""

    def u(x):
        x = np.asarray(x, dtype=float)
        return np.stack([x[..., 1] ** 2, x[..., 0] ** 2 * x[..., 1]], axis=-1)

    def f(x):
        x = np.asarray(x, dtype=float)
        return np.stack([-0.5 * math.pi * (1.0 + 2.0 * x[..., 0]), -0.5 * math.pi * x[..., 1]], axis=-1)

    return ManufacturedProblem(n=2, u_exact=u, f=f, g=u)


def problem_infinity():
    """u = sin(4 pi x1) sin(4 pi x2), f = 32 pi^2 u (Laplacian eigenfunction)."""

    def u(x):
        x = np.asarray(x, dtype=float)
        return np.sin(4.0 * math.pi * x[..., 0]) * np.sin(4.0 * math.pi * x[..., 1])

    def f(x):
        return 32.0 * math.pi ** 2 * u(x)

    return ManufacturedProblem(n=1, u_exact=u, f=f, g=u)
