"""CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It is the checker, never
the product: paper_2207_03921_b200 does not import it.

``liboracle.so`` (nlfem_oracle.c) restates the reference engine operation
for operation (see that file's header for the file:line map) and merges
triplets exactly like ``_merge_triplets`` (assembly.py:137-173) including
numpy's pairwise summation, so on the same inputs it reproduces the
reference's CSR bit for bit.  This is pinned by tests/test_oracle_golden.py
against fixtures generated from the reference itself
(tests/golden/make_golden.py).

Inputs are marshalled by paper_2207_03921_b200.problem.marshal (validation
and tables identical to the reference's bfs_assemble prologue); element
bounds are computed here with numpy exactly as assembly._element_bounds
(:130-134) does.
"""

import ctypes
import os
import subprocess

import numpy as np
from scipy import sparse

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "nlfem_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")


def build(force=False):
    """gcc -O2 -ffp-contract=off -fopenmp (no fused multiply-add, like numba)."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
           "-o", LIB, SRC, "-lm"]
    subprocess.run(cmd, check=True)
    return LIB


_lib = None


class _Prob(ctypes.Structure):
    _fields_ = [
        ("K", ctypes.c_int64), ("V", ctypes.c_int64),
        ("vertices", ctypes.c_void_p), ("elements", ctypes.c_void_p), ("labels", ctypes.c_void_p),
        ("adj_ptr", ctypes.c_void_p), ("adj_idx", ctypes.c_void_p),
        ("centers", ctypes.c_void_p), ("radii", ctypes.c_void_p), ("outer_mask", ctypes.c_void_p),
        ("nc", ctypes.c_int64), ("is_dg", ctypes.c_int64), ("kid", ctypes.c_int64),
        ("s", ctypes.c_double), ("cst", ctypes.c_double), ("delta", ctypes.c_double),
        ("ball_id", ctypes.c_int64), ("path_touch", ctypes.c_int64),
        ("rskip2", ctypes.c_double), ("drop2", ctypes.c_double),
        ("kp0", ctypes.c_double), ("kp1", ctypes.c_double),
        ("symmetric", ctypes.c_int64),
        ("dof_map", ctypes.c_void_p),
        ("n_op", ctypes.c_int64), ("n_ip", ctypes.c_int64),
        ("op", ctypes.c_void_p), ("ow", ctypes.c_void_p), ("oh", ctypes.c_void_p),
        ("ip", ctypes.c_void_p), ("iw", ctypes.c_void_p),
        ("n_sing", ctypes.c_int64 * 3),
        ("sxs", ctypes.c_void_p * 3), ("sys", ctypes.c_void_p * 3), ("sw", ctypes.c_void_p * 3),
        ("shx", ctypes.c_void_p * 3), ("shy", ctypes.c_void_p * 3),
        ("has_lab", ctypes.c_int64), ("lab", ctypes.c_double * 9),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        L.orc_assemble.restype = ctypes.c_void_p
        L.orc_assemble.argtypes = [ctypes.POINTER(_Prob), ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64]
        L.orc_result_nnz.restype = ctypes.c_int64
        L.orc_result_nnz.argtypes = [ctypes.c_void_p]
        L.orc_result_triplets.restype = ctypes.c_int64
        L.orc_result_triplets.argtypes = [ctypes.c_void_p]
        L.orc_result_csr.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 3
        L.orc_result_status.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.orc_result_span_len.restype = ctypes.c_int64
        L.orc_result_span_len.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc_result_span.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4
        L.orc_result_vis.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.orc_result_free.argtypes = [ctypes.c_void_p]
        L.orc_clip_circle.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_void_p]
        L.orc_insert_caps.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        L.orc_clip_square.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_count_visits.argtypes = [ctypes.POINTER(_Prob), ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                       ctypes.c_void_p]
        L.orc_assemble_load.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 4 + [
            ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 5
        _lib = L
    return _lib


def element_bounds(vertices, elements):
    """assembly._element_bounds (:130-134), same numpy expressions."""
    coords = vertices[elements]
    centers = coords.mean(axis=1)
    radii = np.sqrt(((coords - centers[:, None, :]) ** 2).sum(axis=2)).max(axis=1)
    return np.ascontiguousarray(centers), radii


def _p(a):
    return a.ctypes.data


class OracleProblem:
    """Marshalled inputs + element bounds + adjacency, kept alive for ctypes."""

    def __init__(self, inp, adjacency=None):
        self.inp = inp
        self.centers, self.radii = element_bounds(inp.vertices, inp.elements)
        if adjacency is None:
            ptr = np.zeros(inp.elements.shape[0] + 1, dtype=np.int64)
            idx = np.zeros(1, dtype=np.int64)
        else:
            ptr = np.ascontiguousarray(adjacency.ptr, dtype=np.int64)
            idx = np.ascontiguousarray(adjacency.idx, dtype=np.int64)
            if idx.size == 0:
                idx = np.zeros(1, dtype=np.int64)
        self.adj_ptr, self.adj_idx = ptr, idx
        keep = [inp.vertices, inp.elements, inp.labels, inp.outer_mask, inp.dof_map,
                self.centers, self.radii, ptr, idx]
        tabs = [np.ascontiguousarray(t, dtype=np.float64) for t in (inp.op, inp.ow, inp.oh, inp.ip, inp.iw)]
        keep += tabs
        pb = _Prob()
        pb.K, pb.V = inp.elements.shape[0], inp.vertices.shape[0]
        pb.vertices, pb.elements, pb.labels = _p(inp.vertices), _p(inp.elements), _p(inp.labels)
        pb.adj_ptr, pb.adj_idx = _p(ptr), _p(idx)
        pb.centers, pb.radii, pb.outer_mask = _p(self.centers), _p(self.radii), _p(inp.outer_mask)
        pb.nc, pb.is_dg, pb.kid = inp.nc, inp.is_dg, inp.kernel_id
        pb.s, pb.cst, pb.delta = inp.s, inp.scale, inp.delta
        pb.ball_id, pb.path_touch = inp.ball_id, inp.path_touch
        pb.rskip2, pb.drop2, pb.kp0, pb.kp1 = inp.rskip2, inp.drop2, inp.kp0, inp.kp1
        pb.symmetric = inp.symmetric
        pb.has_lab = 1 if len(getattr(inp, "label_scale", ())) else 0
        for i, v in enumerate(getattr(inp, "label_scale", ())):
            pb.lab[i] = v
        pb.dof_map = _p(inp.dof_map)
        pb.n_op, pb.n_ip = inp.op.shape[0], inp.ip.shape[0]
        pb.op, pb.ow, pb.oh, pb.ip, pb.iw = (_p(t) for t in tabs)
        for f, rule in enumerate(inp.rules):
            t = [np.ascontiguousarray(a, dtype=np.float64) for a in (rule.xs, rule.ys, rule.w, rule.hx, rule.hy)]
            keep += t
            pb.n_sing[f] = rule.w.shape[0]
            pb.sxs[f], pb.sys[f], pb.sw[f], pb.shx[f], pb.shy[f] = (_p(a) for a in t)
        self._keep = keep
        self.pb = pb

    def spans(self, k0=0, k1=None, span=64):
        K = self.inp.elements.shape[0]
        k1 = K if k1 is None else k1
        starts = np.arange(k0, k1, span, dtype=np.int64)
        ends = np.minimum(starts + span, k1).astype(np.int64)
        return starts, ends

    def run(self, starts=None, ends=None, brute=False, nthreads=0, raw=False):
        """Engine over the spans + canonical merge.  Returns a dict with the
        CSR (indptr/indices/data over all J rows), status and optionally the
        raw per-span triplets (the reference _chunk outputs)."""
        if starts is None:
            starts, ends = self.spans()
        starts = np.ascontiguousarray(starts, dtype=np.int64)
        ends = np.ascontiguousarray(ends, dtype=np.int64)
        L = lib()
        J = self.inp.n_dofs
        res = L.orc_assemble(ctypes.byref(self.pb), _p(starts), _p(ends), len(starts),
                             1 if brute else 0, int(nthreads), J)
        try:
            nnz = L.orc_result_nnz(res)
            indptr = np.empty(J + 1, dtype=np.int64)
            indices = np.empty(max(nnz, 1), dtype=np.int64)
            data = np.empty(max(nnz, 1), dtype=np.float64)
            L.orc_result_csr(res, _p(indptr), _p(indices), _p(data))
            status = np.empty(7, dtype=np.int64)
            L.orc_result_status(res, _p(status))
            nroots = int((ends - starts).sum())
            vis = np.empty(max(nroots, 1), dtype=np.int64)
            L.orc_result_vis(res, _p(vis), nroots)
            out = {"indptr": indptr, "indices": indices[:nnz], "data": data[:nnz],
                   "err": int(status[0]), "ek": int(status[1]), "el": int(status[2]),
                   "n_inner": int(status[3]), "n_sing_pts": int(status[4]),
                   "epi": int(status[5]), "n_full": int(status[6]),
                   "triplets": int(L.orc_result_triplets(res)), "vis": vis[:nroots]}
            if raw:
                spans = []
                for i in range(len(starts)):
                    n = L.orc_result_span_len(res, i)
                    arrs = [np.empty(max(n, 1), dtype=t) for t in (np.int64, np.int64, np.int64, np.float64)]
                    L.orc_result_span(res, i, *(_p(a) for a in arrs))
                    spans.append(tuple(a[:n] for a in arrs))
                out["spans"] = spans
            return out
        finally:
            L.orc_result_free(res)

    def count_visits(self, k0=0, k1=None, nthreads=0):
        """Per-root EPI (visits passing _visit_pair's reject test, the
        reference's brute traversal) of the roots [k0, k1); 0 for non-outer."""
        K = self.inp.elements.shape[0]
        k1 = K if k1 is None else k1
        vis = np.zeros(max(k1 - k0, 1), dtype=np.int64)
        lib().orc_count_visits(ctypes.byref(self.pb), int(k0), int(k1), int(nthreads), _p(vis))
        return vis[:k1 - k0]

    def matrix(self, **kw):
        r = self.run(**kw)
        J = self.inp.n_dofs
        return sparse.csr_matrix((r["data"], r["indices"], r["indptr"]), shape=(J, J)), r


def assemble(mesh, adjacency, kernel, ansatz, quad=None, rows="all", traversal="bfs", nthreads=0):
    """Oracle counterpart of bfs_assemble: scipy CSR, bit-identical to the reference."""
    from paper_2207_03921_b200.problem import marshal
    inp = marshal(mesh, adjacency, kernel, ansatz, quad, 1, rows, traversal)
    op = OracleProblem(inp, adjacency)
    mat, r = op.matrix(brute=(traversal == "brute"), nthreads=nthreads)
    return mat, r


def band_rows(N, j0, j1, path_touch, nc=1):
    """Rows complete in a band of cell rows [j0, j1) of an N-cell structured
    grid with row-major vertex ids (SURVEY.md 8c band rule): vertex lines
    [j0+1, j1-1] (path 0/1) or [j0+2, j1-1] (path 2, min-owner halo)."""
    lo_line = j0 + (2 if path_touch == 2 else 1)
    hi_line = j1 - 1
    if hi_line < lo_line:
        return 0, 0
    return nc * lo_line * (N + 1), nc * (hi_line + 1) * (N + 1)


def assemble_load(mesh, ansatz, f, quad=None):
    """assembly.assemble_load restated per element (einsum order aside)."""
    from paper_2207_03921_b200.problem import quad_arrays
    from paper_2207_03921_b200.quadrature import QuadratureConfig
    quad = quad or QuadratureConfig()
    op, ow, oh, ip, iw = quad_arrays(quad)
    nc = ansatz.n
    active = np.flatnonzero(mesh.labels != 0)
    coords = mesh.vertices[mesh.elements[active]]
    e1 = coords[:, 1] - coords[:, 0]
    e2 = coords[:, 2] - coords[:, 0]
    pts = (coords[:, None, 0, :] + e1[:, None, :] * op[None, :, 0, None]
           + e2[:, None, :] * op[None, :, 1, None])
    fx = np.ascontiguousarray(np.asarray(f(pts.reshape(-1, 2)), dtype=float).reshape(-1))
    b = np.zeros(ansatz.dof_count)
    V = np.ascontiguousarray(mesh.vertices)
    E = np.ascontiguousarray(mesh.elements, dtype=np.int64)
    Lb = np.ascontiguousarray(mesh.labels, dtype=np.int64)
    D = np.ascontiguousarray(ansatz.dof_map, dtype=np.int64)
    opc, owc, ohc = (np.ascontiguousarray(a) for a in (op, ow, oh))
    lib().orc_assemble_load(E.shape[0], _p(V), _p(E), _p(Lb), _p(D), nc, op.shape[0],
                            _p(opc), _p(owc), _p(ohc), _p(fx), _p(b))
    return b


def assemble_mass(mesh, ansatz):
    """assembly.assemble_mass (:484-506) restated: per active element the
    exact P1 mass block area * (1 + delta_ab) / 12 on each component, summed
    into a J x J CSR.  Areas follow mesh.signed_areas (mesh.py:36-42)."""
    nc = ansatz.n
    active = np.flatnonzero(mesh.labels != 0)
    E = mesh.elements[active]
    p = [mesh.vertices[E[:, i]] for i in range(3)]
    area = 0.5 * ((p[1][:, 0] - p[0][:, 0]) * (p[2][:, 1] - p[0][:, 1])
                  - (p[1][:, 1] - p[0][:, 1]) * (p[2][:, 0] - p[0][:, 0]))
    loc = np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]]) / 12.0
    dk = ansatz.dof_map[active]
    J = ansatz.dof_count
    rows = np.concatenate([(nc * dk[:, a] + c) for c in range(nc) for a in range(3) for b in range(3)])
    cols = np.concatenate([(nc * dk[:, b] + c) for c in range(nc) for a in range(3) for b in range(3)])
    vals = np.concatenate([area * loc[a, b] for c in range(nc) for a in range(3) for b in range(3)])
    m = sparse.coo_matrix((vals, (rows, cols)), shape=(J, J)).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    return m
