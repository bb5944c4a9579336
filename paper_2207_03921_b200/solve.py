"""Dirichlet split, device CG solve and L2 error of the assembled system
(SURVEY.md 8f, next row 1): ``SparseSystem.split`` (assembly.py:102-107)
gives the free-by-free and free-by-constrained blocks; the free block is
solved with ``nlg_cg`` (hand-written warp-per-row SpMV and deterministic
reductions, csrc/nlg.cu) on the GPU.  ``l2_error`` and ``run_study`` are the
harness the reference specifies but does not ship (the L2
error with the 7-point rule on the squared difference, rates
log2(e_prev / e_curr), Tables 2-7 of the paper)."""

import ctypes

import numpy as np

from . import _native
from .errors import ConfigurationError


def cg_device(A, b, x0=None, rtol=1e-12, maxit=None, device=0):
    """Solve A x = b (A: square scipy CSR, symmetric positive definite) with
    conjugate gradients on ``device``.  Returns (x, iterations, relres)."""
    import torch
    A = A.tocsr()
    n = A.shape[0]
    if A.shape != (n, n) or b.shape != (n,):
        raise ConfigurationError(f"cg_device: shapes {A.shape} and {b.shape} do not match")
    dev = f"cuda:{device}"
    ptr = torch.as_tensor(A.indptr.astype(np.int64), device=dev)
    idx = torch.as_tensor(A.indices.astype(np.int32), device=dev)
    val = torch.as_tensor(A.data.astype(np.float64), device=dev)
    rhs = torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64), device=dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev) if x0 is None else \
        torch.as_tensor(np.array(x0, dtype=np.float64), device=dev)
    its = ctypes.c_int32(0)
    res = ctypes.c_double(0.0)
    lib = _native.load_library()
    _native.check(lib.nlg_cg(int(device), int(n), ptr.data_ptr(), idx.data_ptr(), val.data_ptr(), rhs.data_ptr(),
                             x.data_ptr(), float(rtol), int(maxit if maxit is not None else 10 * n + 100),
                             ctypes.byref(its), ctypes.byref(res)), "nlg_cg")
    return x.cpu().numpy(), int(its.value), float(res.value)


def solve_dirichlet(system, b, g=None, rtol=1e-12, maxit=None, device=0):
    """u over all dofs with A_ff u_f = b_f - A_fc g_c and u_c = g_c.

    ``system`` is the SparseSystem of bfs_assemble, ``b`` the load vector
    (assemble_load), ``g`` the Dirichlet data over all dofs (default 0).
    Returns (u, info) with info = {"iterations", "relres"}."""
    free = np.flatnonzero(system.free_mask)
    cons = np.flatnonzero(~system.free_mask)
    a_ff, a_fc = system.split()
    b = np.asarray(b, dtype=np.float64)
    rhs = b[free].copy()
    u = np.zeros(system.matrix.shape[0])
    if g is not None:
        g = np.asarray(g, dtype=np.float64)
        rhs -= a_fc @ g[cons]
        u[cons] = g[cons]
    x, its, res = cg_device(a_ff, rhs, rtol=rtol, maxit=maxit, device=device)
    u[free] = x
    return u, {"iterations": its, "relres": res}


def interpolate(u_exact, mesh, ansatz):
    """Nodal interpolant of ``u_exact`` over all dofs (CG: vertices; DG: the
    element corners), components interleaved like the dofs (nc * base + c)."""
    nc = ansatz.n
    nbase = ansatz.dof_count // nc
    pts = np.zeros((nbase, 2))
    pts[ansatz.dof_map.ravel()] = mesh.vertices[mesh.elements.ravel()]
    vals = np.asarray(u_exact(pts), dtype=float).reshape(nbase, nc)
    return vals.reshape(-1)


def l2_error(coeffs, u_exact, mesh, ansatz, quad=None):
    """sqrt( int_{Omega~} |u_h - u_exact|^2 ) over the active elements, the
    7-point rule applied to the squared difference per element."""
    from .mesh import Label
    from .problem import quad_arrays
    from .quadrature import QuadratureConfig
    op, ow, oh, _, _ = quad_arrays(quad or QuadratureConfig())
    nc = ansatz.n
    act = np.flatnonzero(mesh.labels != Label.INACTIVE)
    xy = mesh.vertices[mesh.elements[act]]                       # (Ka, 3, 2)
    e1, e2 = xy[:, 1] - xy[:, 0], xy[:, 2] - xy[:, 0]
    twoA = e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]
    pts = xy[:, None, 0, :] + e1[:, None, :] * op[None, :, 0, None] + e2[:, None, :] * op[None, :, 1, None]
    c = np.asarray(coeffs, dtype=float).reshape(-1, nc)[ansatz.dof_map[act]]  # (Ka, 3, nc)
    uh = np.einsum("pa,kac->kpc", oh, c)
    ue = np.asarray(u_exact(pts.reshape(-1, 2)), dtype=float).reshape(len(act), op.shape[0], nc)
    sq = ((uh - ue) ** 2).sum(axis=2)
    return float(np.sqrt(np.einsum("p,kp,k->", ow, sq, twoA)))


def run_study(kernel_fn, problem, levels, half_width=0.5, ansatz_kind="cg", quad=None, device=0, rtol=1e-12):
    """Convergence study: for each n_div, the structured
    mesh of (0, half_width)^2 padded by delta, assembly and load on the GPU,
    the Dirichlet solve with g = the interpolant of u_exact, and the L2 error.
    ``kernel_fn()`` returns the KernelSpec.  Rows: dicts with h, dof,
    l2_error, rate (rate = log2(e_prev / e), 0 for the first row)."""
    from .assembly import assemble_load, bfs_assemble, build_ansatz
    from .mesh import build_adjacency_graph, generate_structured_mesh
    kern = kernel_fn()
    rows = []
    for n_div in levels:
        mesh = generate_structured_mesh(half_width, kern.delta, int(n_div))
        ans = build_ansatz(mesh, ansatz_kind, problem.n)
        system = bfs_assemble(mesh, build_adjacency_graph(mesh), kern, ans, quad, device=device)
        b = assemble_load(mesh, ans, problem.f, quad, device=device)
        g = interpolate(problem.g, mesh, ans)
        u, info = solve_dirichlet(system, b, g, rtol=rtol, device=device)
        err = l2_error(u, problem.u_exact, mesh, ans, quad)
        h = float(mesh.h)
        rate = 0.0 if not rows else float(np.log2(rows[-1]["l2_error"] / err))
        rows.append({"n_div": int(n_div), "h": h, "dof": int(np.count_nonzero(ans.free_mask)),
                     "delta": float(kern.delta), "l2_error": err, "rate": rate,
                     "cg_iterations": info["iterations"], "cg_relres": info["relres"]})
    return rows
