"""The five BASELINE.json configurations, as concrete inputs.

Readings follow SURVEY.md Appendix A (seeded synthetic meshes stand in for
the reference's benchmark problems; no dataset is involved):

1. N=32 grid on [-0.1, 1.1]^2, constant kernel 4/(pi delta^4), delta=0.1,
   approxcaps (nocaps also tested), CG n=1, f=1.
2. N=128 grid on [-0.1, 1.1]^2, fractional s=0.4, delta=0.1, approxcaps,
   singular (regularizing) path for touching pairs, f=1.
3. N=256 grid on [-0.05, 1.05]^2, peridynamic 3/delta^3, delta=0.05, nocaps,
   CG n=2 (6x6 element blocks), body force (0, -1); ``transform=True`` gives
   the singular-rule variant.
4. N=2048 grid on [-0.02, 1.02]^2, constant kernel, delta=0.02, approxcaps.
5. L-shape: N=512 grid on [-0.1, 1.1]^2 minus cells with centre x, y > 0.6,
   perturb(amplitude=0.2, seed=0), all DOMAIN (pure Neumann), nonsymmetric
   (1 + 0.5 x_1) 4/(pi delta^4), delta=0.1, approxcaps.
"""

from dataclasses import dataclass, field

import numpy as np

from .assembly import build_ansatz
from .kernels import affine_kernel, constant_kernel, fractional_kernel, peridynamic_kernel
from .mesh import build_adjacency_graph, grid_mesh, lshape_mesh, perturb
from .quadrature import QuadratureConfig


@dataclass
class Config:
    name: str
    mesh: object
    kernel: object
    ansatz: object
    quad: object
    f: object
    grid_n: int
    _adjacency: object = field(default=None, repr=False)

    @property
    def adjacency(self):
        if self._adjacency is None:
            self._adjacency = build_adjacency_graph(self.mesh)
        return self._adjacency

    def describe(self):
        return {"workload": self.name, "K": int(self.mesh.n_elements), "J": int(self.ansatz.dof_count),
                "kernel_id": int(self.kernel.builtin_id), "ball": self.kernel.ball,
                "delta": float(self.kernel.delta), "nc": int(self.ansatz.n)}


def _one(x):
    return np.ones(x.shape[0])


def _body(x):
    return np.column_stack([np.zeros(x.shape[0]), -np.ones(x.shape[0])])


def build(n, ball=None, transform=False, grid_n=None):
    """Config ``n`` (1-5).  ``ball`` overrides the ball, ``grid_n`` the grid
    resolution (reduced-size parity cases of the same construction)."""
    if n == 1:
        N = grid_n or 32
        mesh = grid_mesh(N, -0.1, 1.1, delta=0.1)
        kern = constant_kernel(0.1, ball or "approxcaps")
        return Config(f"cfg1_N{N}_const_{kern.ball}", mesh, kern, build_ansatz(mesh), QuadratureConfig(), _one, N)
    if n == 2:
        N = grid_n or 128
        mesh = grid_mesh(N, -0.1, 1.1, delta=0.1)
        kern = fractional_kernel(0.4, 0.1, ball or "approxcaps")
        return Config(f"cfg2_N{N}_frac0.4_{kern.ball}", mesh, kern, build_ansatz(mesh), QuadratureConfig(), _one, N)
    if n == 3:
        N = grid_n or 256
        mesh = grid_mesh(N, -0.05, 1.05, delta=0.05)
        kern = peridynamic_kernel(0.05, ball or "nocaps")
        quad = QuadratureConfig(weak_singular="transform" if transform else "avoid")
        tag = "transform" if transform else "avoid"
        return Config(f"cfg3_N{N}_peri_{kern.ball}_{tag}", mesh, kern, build_ansatz(mesh, "cg", 2), quad, _body, N)
    if n == 4:
        N = grid_n or 2048
        mesh = grid_mesh(N, -0.02, 1.02, delta=0.02)
        kern = constant_kernel(0.02, ball or "approxcaps")
        return Config(f"cfg4_N{N}_const_{kern.ball}", mesh, kern, build_ansatz(mesh), QuadratureConfig(), _one, N)
    if n == 5:
        N = grid_n or 512
        mesh = perturb(lshape_mesh(N), amplitude=0.2, seed=0)
        kern = affine_kernel(0.1, 0.5, ball=ball or "approxcaps")
        return Config(f"cfg5_L{N}_affine_{kern.ball}", mesh, kern, build_ansatz(mesh), QuadratureConfig(), _one, N)
    raise ValueError(f"unknown config {n}")
