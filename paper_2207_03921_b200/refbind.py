"""Reference-side binding: the ctypes stub of INTEGRATION.md §2, as code.

A maintainer of nlfem routes ``bfs_assemble``'s compiled-engine branch
through ``libnlg.so`` by handing this module the two tuples the reference
already builds for ``_engine._chunk`` (``/root/reference/pkg/src/nlfem/
assembly.py:249-264``)::

    args  = (vertices, elements, labels, adj_ptr, adj_idx, centers, radii, outer,
             nc, is_dg, builtin_id, s, scale, delta, ball_id, path_touch,
             rskip2, drop2, dof_map, op, ow, oh, ip, iw)
    sargs = (xs, ys, w, hx, hy) of the identical, edge and vertex rules

and replacing the span thread pool + ``_merge_triplets`` (:245-296) with::

    matrix = refbind.assemble_engine_args(args, sargs, ansatz.dof_count)

``problem_from_engine_args`` is the marshalling alone (no GPU needed); it
fills the ``nlg_problem`` struct of include/nlg.h field by field from those
tuples.  The adjacency, centres and radii the reference computed are not
needed: the device recomputes the bounds and searches a grid.
"""

import ctypes

import numpy as np
from scipy import sparse

from . import _native
from .errors import ConfigurationError, NumericalError

ENGINE_ARGS = ("vertices", "elements", "labels", "adj_ptr", "adj_idx", "centers", "radii", "outer", "nc",
               "is_dg", "builtin_id", "s", "scale", "delta", "ball_id", "path_touch", "rskip2", "drop2",
               "dof_map", "op", "ow", "oh", "ip", "iw")


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def problem_from_engine_args(args, sargs, J):
    """(nlg_problem, keep-alive list) from the reference's _chunk argument tuples."""
    if len(args) != len(ENGINE_ARGS) or len(sargs) != 15:
        raise ConfigurationError("expected the 24 _engine._chunk arguments and 15 singular-rule tables")
    a = dict(zip(ENGINE_ARGS, args))
    if int(a["builtin_id"]) < 0:
        raise ConfigurationError("the compiled-engine arguments carry a built-in kernel id >= 0")
    keep = []
    pb = _native.Problem()
    verts, elems = _c(a["vertices"], np.float64), _c(a["elements"], np.int64)
    labels, outer, dof_map = _c(a["labels"], np.int64), _c(a["outer"], np.int64), _c(a["dof_map"], np.int64)
    keep += [verts, elems, labels, outer, dof_map]
    pb.n_vertices, pb.n_elements = verts.shape[0], elems.shape[0]
    pb.vertices, pb.elements, pb.labels = verts.ctypes.data, elems.ctypes.data, labels.ctypes.data
    pb.outer_mask, pb.dof_map, pb.n_dofs = outer.ctypes.data, dof_map.ctypes.data, int(J)
    pb.nc, pb.is_dg, pb.kernel_id = int(a["nc"]), int(a["is_dg"]), int(a["builtin_id"])
    pb.symmetric = 1  # the reference's compiled kernels (ids 0-2) are symmetric
    pb.ball_id, pb.path_touch = int(a["ball_id"]), int(a["path_touch"])
    pb.s, pb.scale, pb.delta = float(a["s"]), float(a["scale"]), float(a["delta"])
    pb.rskip2, pb.drop2, pb.kp0, pb.kp1 = float(a["rskip2"]), float(a["drop2"]), 0.0, 0.0
    tabs = [_c(a[n], np.float64) for n in ("op", "ow", "oh", "ip", "iw")]
    keep += tabs
    pb.n_outer, pb.n_inner = tabs[0].shape[0], tabs[3].shape[0]
    pb.op, pb.ow, pb.oh, pb.ip, pb.iw = (t.ctypes.data for t in tabs)
    for f in range(3):  # identical, edge, vertex
        t = [_c(x, np.float64) for x in sargs[5 * f:5 * f + 5]]
        keep += t
        pb.n_sing[f] = t[2].shape[0]
        pb.sxs[f], pb.sys[f], pb.sw[f], pb.shx[f], pb.shy[f] = (x.ctypes.data for x in t)
    pb.inputs_on_device = 0
    return pb, keep


def assemble_engine_args(args, sargs, J, *, device=0, row_range=None, traversal="bfs"):
    """The J x J (or row-block) scipy CSR the reference's merge would return."""
    lib = _native.load_library()
    pb, keep = problem_from_engine_args(args, sargs, J)
    lo, hi = (0, int(J)) if row_range is None else (int(row_range[0]), int(row_range[1]))
    plan = ctypes.c_void_p()
    _native.check(lib.nlg_plan_create(int(device), ctypes.byref(pb), None, ctypes.byref(plan)), "nlg_plan_create")
    sink = _native.OutputSink(True, device)
    st = _native.Stats()
    try:
        rc = lib.nlg_assemble(plan, lo, hi, 1, sink.callback, None, 0, ctypes.byref(st))
    finally:
        lib.nlg_plan_destroy(plan)
    if rc == _native.NLG_ERR_NUMERICAL and st.err_k >= 0:
        k, l = int(st.err_k), int(st.err_l)
        if traversal == "bfs" and st.err_self_k == k:
            l = k
        raise NumericalError(f"nonfinite local contribution for element pair ({k}, {l})")
    _native.check(rc, "nlg_assemble")
    del keep
    return sparse.csr_matrix((sink.array(2, np.float64, st.nnz), sink.array(1, np.int32, st.nnz),
                              sink.array(0, np.int64, hi - lo + 1)), shape=(hi - lo, int(J)))
