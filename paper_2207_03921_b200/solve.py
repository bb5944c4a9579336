"""Dirichlet split and a device CG solve of the assembled system (SURVEY.md
8f, next row 1): ``SparseSystem.split`` (assembly.py:102-107) gives the
free-by-free and free-by-constrained blocks; the free block is solved with
``nlg_cg`` (hand-written warp-per-row SpMV and deterministic reductions,
csrc/nlg.cu) on the GPU."""

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
