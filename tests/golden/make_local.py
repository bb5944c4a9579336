"""Golden per-pair blocks from the REFERENCE's local_contribution
(assembly.py:327-448), for tests/test_gpu_local.py.

    python tests/golden/make_local.py

For a few of the fixture cases (meshes and kernels as make_golden.py builds
them), a deterministic sample of ordered element pairs -- identical,
edge- and vertex-touching, fully inside, near the ball's rim, far -- is
evaluated by the reference; blocks, rows and the pairs are stored in
tests/golden/local_<case>.npz.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as G  # noqa: E402  (the reference on sys.path, the cases)

from nlfem import assembly as A  # noqa: E402
from nlfem.quadrature import QuadratureConfig  # noqa: E402

CASES = ["cfg1_nocaps", "frac_s04_approx_pert", "peri_nocaps_avoid", "peri_approx_transform", "const_inf_pert",
         "lshape16_affine", "frac_s04_nocaps_dg"]


def sample_pairs(mesh, delta, rng, n=24):
    E, V = mesh.elements, mesh.vertices
    c = V[E].mean(axis=1)
    K = E.shape[0]
    act = np.flatnonzero(mesh.labels != 0)
    pairs = set()
    roots = rng.choice(act, size=min(6, act.size), replace=False)
    for k in roots:
        k = int(k)
        pairs.add((k, k))
        touch = [int(l) for l in act if l != k and np.intersect1d(E[k], E[l]).size > 0]
        for l in touch[:3]:
            pairs.add((k, l))
        d = np.linalg.norm(c[act] - c[k], axis=1)
        for lo, hi in ((0.2 * delta, 0.6 * delta), (0.85 * delta, 1.15 * delta), (1.3 * delta, 2.0 * delta)):
            cand = act[(d > lo) & (d < hi)]
            if cand.size:
                pairs.add((k, int(rng.choice(cand))))
    return sorted(pairs)[: max(n, 0) or None]


def main():
    cases = G.cases()
    for name in CASES:
        mesh, kern, spec, kind, n, quad, rows, f = cases[name]
        ans = A.build_ansatz(mesh, kind, n)
        q = QuadratureConfig(**quad)
        rng = np.random.default_rng(11)
        pairs = sample_pairs(mesh, kern.delta, rng, n=40)
        blocks, rws, dims = [], [], []
        nb = 6 * n
        for k, l in pairs:
            ls = A.local_contribution(k, l, kern, ans, q, mesh)
            d = ls.block.shape[0]
            b = np.zeros((nb, nb))
            b[:d, :d] = ls.block
            r = np.zeros(nb, dtype=np.int64)
            r[:d] = ls.rows
            blocks.append(b)
            rws.append(r)
            dims.append(d)
        np.savez_compressed(os.path.join(HERE, f"local_{name}.npz"), pairs=np.array(pairs, dtype=np.int64),
                            blocks=np.array(blocks), rows=np.array(rws), dims=np.array(dims, dtype=np.int32))
        print(name, len(pairs), "pairs")


if __name__ == "__main__":
    main()
