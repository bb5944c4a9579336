"""Generate golden fixtures by running the REFERENCE (not this repo's code).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each case builds its mesh with the reference's own generators
(nlfem.mesh.generate_structured_mesh / perturb) or, for the BASELINE
configs, with the Appendix-A grid fed to nlfem.mesh.Mesh; assembles with
nlfem.assembly.bfs_assemble (numba engine for built-in kernels, the
interpreted engine for the nonsymmetric callable kernel) and
nlfem.assembly.assemble_load; and stores inputs + outputs in
tests/golden/<case>.npz.  The fixtures travel with the repo; the GPU box
never needs /root/reference.
"""

import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from nlfem import assembly as A  # noqa: E402
from nlfem import kernels as KR  # noqa: E402
from nlfem import mesh as M  # noqa: E402
from nlfem.quadrature import QuadratureConfig  # noqa: E402

from paper_2207_03921_b200 import mesh as mine  # noqa: E402  (Appendix-A grid only)


def grid(N, lo, hi):
    m = mine.grid_mesh(N, lo, hi)
    return M.Mesh(m.vertices, m.elements, m.labels)


def lshape(N):
    m = mine.lshape_mesh(N)
    return M.perturb(M.Mesh(m.vertices, m.elements, m.labels), amplitude=0.2, seed=0)


def const_kernel(delta, ball, scale):
    return KR.KernelSpec(delta=delta, s=-1.0, n=1, symmetric=True, ball=ball,
                         value=lambda x, y, lx=1, ly=1: np.array([[scale]]),
                         builtin_id=2, scale=scale)


def affine_kernel(delta, alpha, c, ball):
    return KR.KernelSpec(delta=delta, s=-1.0, n=1, symmetric=False, ball=ball,
                         value=lambda x, y, lx=1, ly=1: np.array([[(1.0 + alpha * x[0]) * c]]))


def labeled(base, tab2):
    """Label-dependent kernel as the reference takes it: a Python callable
    (builtin_id -1, interpreted engine) value = T[label_x][label_y] * base."""
    T = np.zeros((3, 3))
    T[1:, 1:] = np.asarray(tab2, dtype=float)
    T = [[float(v) for v in row] for row in T]
    bval = base.value
    return KR.KernelSpec(delta=base.delta, s=base.s, n=base.n, symmetric=True, ball=base.ball,
                         value=lambda x, y, lx=1, ly=1: T[int(lx)][int(ly)] * bval(x, y))


def cases():
    d = 0.1
    c1 = 4.0 / (math.pi * d ** 4)
    out = {}
    cfg1 = grid(32, -0.1, 1.1)
    out["cfg1_approxcaps"] = (cfg1, const_kernel(d, "approxcaps", c1),
                              {"id": 2, "ball": "approxcaps", "delta": d, "scale": c1}, "cg", 1, {}, "all", "one")
    out["cfg1_nocaps"] = (cfg1, const_kernel(d, "nocaps", c1),
                          {"id": 2, "ball": "nocaps", "delta": d, "scale": c1}, "cg", 1, {}, "all", "one")
    small = M.perturb(M.generate_structured_mesh(1.0, 0.2, 10), amplitude=0.2, seed=3)
    out["frac_s04_approx_pert"] = (small, KR.fractional_kernel(0.4, 0.2, "approxcaps"),
                                   {"id": 0, "s": 0.4, "ball": "approxcaps", "delta": 0.2}, "cg", 1, {}, "all", "x")
    out["frac_s04_nocaps_dg"] = (M.generate_structured_mesh(1.0, 0.2, 5), KR.fractional_kernel(0.4, 0.2, "nocaps"),
                                 {"id": 0, "s": 0.4, "ball": "nocaps", "delta": 0.2}, "dg", 1, {}, "all", "x")
    out["frac_s07_infinity"] = (small, KR.fractional_kernel(0.7, 0.2, "infinity"),
                                {"id": 0, "s": 0.7, "ball": "infinity", "delta": 0.2}, "cg", 1, {}, "domain", "x")
    out["peri_nocaps_avoid"] = (small, KR.peridynamic_kernel(0.2, "nocaps"),
                                {"id": 1, "ball": "nocaps", "delta": 0.2}, "cg", 2, {}, "all", "body")
    out["peri_approx_transform"] = (small, KR.peridynamic_kernel(0.2, "approxcaps"),
                                    {"id": 1, "ball": "approxcaps", "delta": 0.2}, "cg", 2,
                                    {"weak_singular": "transform"}, "all", "body")
    out["const_inf_pert"] = (small, KR.constant_kernel_infinity(0.2),
                             {"id": 2, "ball": "infinity", "delta": 0.2, "scale": 3.0 / (4.0 * 0.2 ** 4)},
                             "cg", 1, {}, "all", "x")
    out["const_allfull"] = (M.perturb(M.generate_structured_mesh(1.0, 0.0, 6), amplitude=0.2, seed=1),
                            const_kernel(5.0, "approxcaps", 1.0),
                            {"id": 2, "ball": "approxcaps", "delta": 5.0, "scale": 1.0}, "cg", 1, {}, "all", "one")
    lm = lshape(16)
    out["lshape16_affine"] = (lm, affine_kernel(0.1, 0.5, c1, "approxcaps"),
                              {"id": 3, "ball": "approxcaps", "delta": 0.1, "alpha": 0.5, "scale": c1},
                              "cg", 1, {}, "all", "one")
    out["lshape16_const"] = (lm, const_kernel(0.1, "approxcaps", c1),
                             {"id": 2, "ball": "approxcaps", "delta": 0.1, "scale": c1}, "cg", 1, {}, "all", "one")
    # label-dependent kernels (interface coefficients per pair of subdomains)
    t1, t2, t3 = [[1.0, 0.5], [0.5, 2.0]], [[1.0, 0.25], [0.25, 3.0]], [[1.0, 2.0], [2.0, 0.5]]
    out["frac_s04_labels"] = (small, labeled(KR.fractional_kernel(0.4, 0.2, "approxcaps"), t1),
                              {"id": 0, "s": 0.4, "ball": "approxcaps", "delta": 0.2, "labels": t1},
                              "cg", 1, {}, "all", "x")
    out["lshape16_const_labels"] = (lm, labeled(const_kernel(0.1, "approxcaps", c1), t2),
                                    {"id": 2, "ball": "approxcaps", "delta": 0.1, "scale": c1, "labels": t2},
                                    "cg", 1, {}, "all", "one")
    out["peri_nocaps_labels"] = (small, labeled(KR.peridynamic_kernel(0.2, "nocaps"), t3),
                                 {"id": 1, "ball": "nocaps", "delta": 0.2, "labels": t3}, "cg", 2, {}, "all", "body")
    return out


FUNCS = {
    "one": lambda x: np.ones(x.shape[0]),
    "x": lambda x: x[:, 0] * x[:, 1] + 1.0,
    "body": lambda x: np.column_stack([np.zeros(x.shape[0]), -np.ones(x.shape[0])]),
}


def main(only=None):
    for name, (mesh, kernel, kspec, kind, n, qkw, rows, fname) in cases().items():
        if only and name not in only:
            continue
        t0 = time.time()
        adj = M.build_adjacency_graph(mesh)
        ans = A.build_ansatz(mesh, kind, n)
        quad = QuadratureConfig(**qkw)
        sysm = A.bfs_assemble(mesh, adj, kernel, ans, quad, n_threads=8, rows=rows)
        mat = sysm.matrix
        b = A.assemble_load(mesh, ans, FUNCS[fname], quad)
        spec = {"kernel": kspec, "ansatz": kind, "n": n, "quad": qkw, "rows": rows, "f": fname}
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            vertices=mesh.vertices, elements=mesh.elements, labels=mesh.labels,
            indptr=mat.indptr.astype(np.int64), indices=mat.indices.astype(np.int64), data=mat.data,
            b=b, free_mask=sysm.free_mask, spec=np.array(json.dumps(spec)))
        print(f"{name}: K={mesh.n_elements} J={ans.dof_count} nnz={mat.nnz} "
              f"|A|_F={np.linalg.norm(mat.data):.16g} ({time.time() - t0:.1f}s)")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
