"""Load tests/golden/*.npz fixtures (made by make_golden.py from the
reference) into this package's host types."""

import glob
import json
import os

import numpy as np
from scipy import sparse

from paper_2207_03921_b200 import kernels as KR
from paper_2207_03921_b200.assembly import build_ansatz
from paper_2207_03921_b200.mesh import Mesh, build_adjacency_graph
from paper_2207_03921_b200.quadrature import QuadratureConfig

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

FUNCS = {
    "one": lambda x: np.ones(x.shape[0]),
    "x": lambda x: x[:, 0] * x[:, 1] + 1.0,
    "body": lambda x: np.column_stack([np.zeros(x.shape[0]), -np.ones(x.shape[0])]),
}


def names():
    """The whole-assembly fixtures (local_*.npz hold per-pair blocks)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith("local_"))


def kernel_from_spec(k):
    kid, ball, delta = k["id"], k["ball"], k["delta"]
    if kid == 0:
        base = KR.fractional_kernel(k["s"], delta, ball)
    elif kid == 1:
        base = KR.peridynamic_kernel(delta, ball)
    elif kid == 2:
        base = KR.constant_kernel(delta, ball, scale=k["scale"])
    else:
        base = KR.affine_kernel(delta, k["alpha"], k["scale"], ball)
    return KR.label_scaled_kernel(base, k["labels"]) if "labels" in k else base


class Case:
    def __init__(self, name):
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.name = name
        self.spec = json.loads(str(z["spec"]))
        self.mesh = Mesh(z["vertices"], z["elements"], z["labels"])
        self.adjacency = build_adjacency_graph(self.mesh)
        self.kernel = kernel_from_spec(self.spec["kernel"])
        self.ansatz = build_ansatz(self.mesh, self.spec["ansatz"], self.spec["n"])
        self.quad = QuadratureConfig(**self.spec["quad"])
        self.rows = self.spec["rows"]
        self.f = FUNCS[self.spec["f"]]
        J = self.ansatz.dof_count
        self.matrix = sparse.csr_matrix((z["data"], z["indices"], z["indptr"]), shape=(J, J))
        self.b = z["b"]
        self.free_mask = z["free_mask"]

    def args(self):
        return (self.mesh, self.adjacency, self.kernel, self.ansatz, self.quad)


def rel_fro(a, b):
    """||A - B||_F / ||B||_F over the union pattern."""
    d = (a - b).tocsr()
    nb = np.linalg.norm(b.data) if b.nnz else 1.0
    return np.linalg.norm(d.data) / (nb if nb else 1.0)


def same_pattern(a, b):
    a = a.tocsr()
    b = b.tocsr()
    a.sort_indices()
    b.sort_indices()
    return np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)


def sample_vertices(mesh, n=40, seed=0, extra=()):
    """Deterministic vertex sample: corners of the bounding box plus n random."""
    rng = np.random.default_rng(seed)
    V = mesh.vertices
    picks = set(int(i) for i in extra)
    for fx in (np.argmin, np.argmax):
        picks.add(int(fx(V[:, 0] + V[:, 1])))
        picks.add(int(fx(V[:, 0] - V[:, 1])))
    picks.update(int(i) for i in rng.choice(mesh.n_vertices, size=min(n, mesh.n_vertices), replace=False))
    return np.array(sorted(picks), dtype=np.int64)


def oracle_rows(inp, adjacency, mesh, verts, nthreads=0):
    """CPU-oracle CSR rows of the given vertices (all components).

    Runs the reference restatement only on the outer elements that reach
    those rows: elements containing a vertex, plus (touching-pair owner rule
    on the regularizing path) every element touching one of them.
    """
    from oracle import oracle
    E = mesh.elements
    inc = np.isin(E, verts).any(axis=1)
    roots = set(np.flatnonzero(inc).tolist())
    if inp.path_touch == 2:
        vs = np.unique(E[inc])
        roots |= set(np.flatnonzero(np.isin(E, vs).any(axis=1)).tolist())
    roots = np.array(sorted(roots), dtype=np.int64)
    op = oracle.OracleProblem(inp, adjacency)
    r = op.run(starts=roots, ends=roots + 1, nthreads=nthreads)
    J = inp.n_dofs
    full = sparse.csr_matrix((r["data"], r["indices"], r["indptr"]), shape=(J, J))
    rows = (inp.nc * verts[:, None] + np.arange(inp.nc)[None, :]).ravel()
    return rows, full[rows]
