"""The drop-in boundary against the reference's own objects (CPU, no GPU).

* ``bfs_assemble`` / ``marshal`` accept kernels, meshes, adjacency graphs,
  ansatz spaces and quadrature configs built by the reference's factories
  (``nlfem.kernels`` etc.) and marshal them exactly like this package's
  restated types (assembly.py:212-264);
* the exceptions are the reference's classes (subclasses), so callers
  catching ``nlfem.errors.*`` keep working (errors.py:4-13);
* the reference-side stub of INTEGRATION.md (``refbind``) marshals the very
  argument tuples the reference hands to ``_engine._chunk`` into the
  ``nlg_problem`` struct of include/nlg.h, field for field.
"""

import numpy as np
import pytest

from paper_2207_03921_b200 import (ConfigurationError, NumericalError, bfs_assemble, build_adjacency_graph,
                                   build_ansatz, grid_mesh, perturb)
from paper_2207_03921_b200 import kernels as K
from paper_2207_03921_b200.problem import marshal
from paper_2207_03921_b200.quadrature import QuadratureConfig


def _ref_objects(reference, kind="frac"):
    import nlfem.assembly as RA
    import nlfem.kernels as RK
    import nlfem.mesh as RM
    import nlfem.quadrature as RQ
    m = perturb(grid_mesh(10, -0.2, 1.2, delta=0.2), amplitude=0.2, seed=3)
    rmesh = RM.Mesh(m.vertices, m.elements, m.labels)
    radj = RM.build_adjacency_graph(rmesh)
    if kind == "frac":
        rk, ok = RK.fractional_kernel(0.4, 0.2, "approxcaps"), K.fractional_kernel(0.4, 0.2, "approxcaps")
        n = 1
    elif kind == "peri":
        rk, ok = RK.peridynamic_kernel(0.2, "nocaps"), K.peridynamic_kernel(0.2, "nocaps")
        n = 2
    else:
        rk, ok = RK.constant_kernel_infinity(0.2), K.constant_kernel_infinity(0.2)
        n = 1
    rans = RA.build_ansatz(rmesh, "cg", n)
    rquad = RQ.QuadratureConfig(weak_singular="transform" if kind == "peri" else "avoid")
    ours = (m, build_adjacency_graph(m), ok, build_ansatz(m, "cg", n),
            QuadratureConfig(weak_singular=rquad.weak_singular))
    return (rmesh, radj, rk, rans, rquad), ours


def _same_inputs(a, b):
    for f in a.__dataclass_fields__:
        x, y = getattr(a, f), getattr(b, f)
        if f == "rules":
            for ra, rb in zip(x, y):
                for t in ("xs", "ys", "w", "hx", "hy"):
                    assert np.array_equal(getattr(ra, t), getattr(rb, t)), (f, t)
        elif isinstance(x, np.ndarray):
            assert x.dtype == y.dtype and np.array_equal(x, y), f
        else:
            assert x == y, f


@pytest.mark.parametrize("kind", ["frac", "peri", "const_inf"])
def test_reference_objects_marshal_like_ours(reference, kind):
    theirs, ours = _ref_objects(reference, kind)
    _same_inputs(marshal(*theirs), marshal(*ours))


def test_exceptions_are_the_reference_classes(reference):
    import nlfem.errors as RE

    from paper_2207_03921_b200 import errors
    if not errors.REFERENCE_LINKED:
        pytest.skip("package imported before the reference was importable")
    assert issubclass(ConfigurationError, RE.ConfigurationError) and issubclass(ConfigurationError, ValueError)
    assert issubclass(NumericalError, RE.NumericalError) and issubclass(NumericalError, RuntimeError)
    from paper_2207_03921_b200 import MeshFormatError
    assert issubclass(MeshFormatError, RE.MeshFormatError) and issubclass(MeshFormatError, ConfigurationError)
    theirs, _ = _ref_objects(reference)
    # validation happens before any device work: no GPU needed
    with pytest.raises(RE.ConfigurationError, match="rows must be"):
        bfs_assemble(*theirs, rows="some")
    with pytest.raises(RE.ConfigurationError, match="traversal must be"):
        bfs_assemble(*theirs, traversal="dfs")
    with pytest.raises(RE.ConfigurationError, match="kernel must be a KernelSpec"):
        bfs_assemble(theirs[0], theirs[1], object(), theirs[3])


def test_reference_callable_kernel_rejected(reference):
    import nlfem.kernels as RK
    theirs, _ = _ref_objects(reference)
    k = RK.KernelSpec(delta=0.2, s=-1.0, n=1, symmetric=False, ball="approxcaps",
                      value=lambda x, y, lx, ly: np.array([[1.0 + 0.5 * x[0]]]))
    with pytest.raises(ConfigurationError, match="built-in kernels only"):
        bfs_assemble(theirs[0], theirs[1], k, theirs[3])


def engine_args_like_reference(inp, adjacency, centers, radii):
    """The tuple the reference builds at assembly.py:249-260 (from marshal's fields)."""
    return ((inp.vertices, inp.elements, inp.labels, adjacency.ptr, adjacency.idx, centers, radii,
             inp.outer_mask, inp.nc, inp.is_dg, inp.kernel_id, inp.s, inp.scale, inp.delta, inp.ball_id,
             inp.path_touch, inp.rskip2, inp.drop2, inp.dof_map, inp.op, inp.ow, inp.oh, inp.ip, inp.iw),
            tuple(a for r in inp.rules for a in (r.xs, r.ys, r.w, r.hx, r.hy)))


def _capture_engine_args(monkeypatch, theirs):
    """Run the reference's bfs_assemble with _engine._chunk replaced by a
    recorder: returns the exact (args, sargs) it hands the engine."""
    import nlfem._engine as RE_
    import nlfem.assembly as RA
    seen = []

    def chunk(k0, k1, brute, *rest):
        seen.append(rest)
        z = np.zeros(0, dtype=np.int64)
        return z, z, z, np.zeros(0), np.zeros(k1 - k0, dtype=np.int64), 0, -1, -1

    monkeypatch.setattr(RE_, "_chunk", chunk)
    RA.bfs_assemble(*theirs, traversal="brute")
    rest = seen[0]
    return rest[:24], rest[24:]


@pytest.mark.parametrize("kind", ["frac", "peri"])
def test_integration_stub_marshals_reference_engine_args(reference, monkeypatch, kind):
    from paper_2207_03921_b200 import _native, refbind
    theirs, ours = _ref_objects(reference, kind)
    args, sargs = _capture_engine_args(monkeypatch, theirs)
    assert len(args) == 24 and len(sargs) == 15
    J = theirs[3].dof_count
    pb, keep = refbind.problem_from_engine_args(args, sargs, J)
    # the same struct this package's own path builds from its own types
    inp = marshal(*ours)
    mine, keep2 = refbind.problem_from_engine_args(*engine_args_like_reference(
        inp, ours[1], np.zeros((1, 2)), np.zeros(1)), J)
    for name, ctype in _native.Problem._fields_:
        a, b = getattr(pb, name), getattr(mine, name)
        if name in ("vertices", "elements", "labels", "outer_mask", "dof_map", "op", "ow", "oh", "ip", "iw",
                    "sxs", "sys", "sw", "shx", "shy"):
            continue  # pointers: compared by content below
        if hasattr(a, "__len__"):
            assert list(a) == list(b), name
        else:
            assert a == b, name
    def arr(ptr, n, dt):
        return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(dt)), shape=(n,)).copy()
    import ctypes
    K_, V_ = pb.n_elements, pb.n_vertices
    for name, n, dt in (("vertices", 2 * V_, ctypes.c_double), ("elements", 3 * K_, ctypes.c_int64),
                        ("labels", K_, ctypes.c_int64), ("outer_mask", K_, ctypes.c_int64),
                        ("dof_map", 3 * K_, ctypes.c_int64), ("op", 14, ctypes.c_double),
                        ("ow", 7, ctypes.c_double), ("oh", 21, ctypes.c_double), ("ip", 14, ctypes.c_double),
                        ("iw", 7, ctypes.c_double)):
        assert np.array_equal(arr(getattr(pb, name), n, dt), arr(getattr(mine, name), n, dt)), name
    for f in range(3):
        n = pb.n_sing[f]
        for name, m in (("sxs", 2), ("sys", 2), ("sw", 1), ("shx", 3), ("shy", 3)):
            assert np.array_equal(arr(getattr(pb, name)[f], m * n, ctypes.c_double),
                                  arr(getattr(mine, name)[f], m * n, ctypes.c_double)), (name, f)
