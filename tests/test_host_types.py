"""Host-side restatements vs the reference (skipped where the reference tree
is absent) and vs the SPEC's known answers; plus the C ABI export check."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_2207_03921_b200 import (ConfigurationError, Label, Mesh, QuadratureConfig, build_adjacency_graph,
                                   build_ansatz, dispatch, fractional_kernel, gauss_legendre,
                                   generate_structured_mesh, grid_mesh, lshape_mesh, peridynamic_kernel,
                                   perturb, rule_7point, singular_rule)
from paper_2207_03921_b200.geometry import PairClass
from paper_2207_03921_b200.problem import marshal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_singular_rules_bitwise_equal_reference(reference):
    from nlfem import quadrature as rq
    for kind in ("identical", "edge", "vertex"):
        for n in (2, 3, 5):
            a, b = rq.singular_rule(kind, n), singular_rule(kind, n)
            for f in ("xs", "ys", "w", "hx", "hy"):
                assert np.array_equal(getattr(a, f), getattr(b, f)), (kind, n, f)


def test_rule_exactness():
    # 7-point rule exact for degree <= 3; Gauss n=5 exact for t^9
    pts, w = rule_7point()
    assert abs(w.sum() - 0.5) < 1e-15
    for i in range(4):
        for j in range(4 - i):
            exact = math.factorial(i) * math.factorial(j) / math.factorial(i + j + 2)
            assert abs((w * pts[:, 0] ** i * pts[:, 1] ** j).sum() - exact) < 1e-15
    g, gw = gauss_legendre(5)
    assert abs((gw * g ** 9).sum() - 0.1) < 1e-14
    for kind in ("identical", "edge", "vertex"):
        assert abs(singular_rule(kind, 5).w.sum() - 0.25) < 1e-14


def test_dispatch_table():
    assert dispatch(-1.0, PairClass.IDENTICAL).value == "standard"
    assert dispatch(-0.5, PairClass.IDENTICAL).value == "avoid-diagonal"
    assert dispatch(-0.5, PairClass.IDENTICAL, "transform").value == "regularizing"
    assert dispatch(0.4, PairClass.EDGE_TOUCHING).value == "regularizing"
    assert dispatch(0.4, PairClass.DISJOINT).value == "standard"
    with pytest.raises(ConfigurationError):
        dispatch(1.0, PairClass.DISJOINT)


def test_perturb_and_generators_match_reference(reference):
    import nlfem.mesh as rm
    r = rm.perturb(rm.generate_structured_mesh(1.0, 0.2, 10), amplitude=0.2, seed=3)
    m = perturb(generate_structured_mesh(1.0, 0.2, 10), amplitude=0.2, seed=3)
    assert np.array_equal(r.vertices, m.vertices)
    assert np.array_equal(r.elements, m.elements)
    assert np.array_equal(r.labels, m.labels)
    assert r.h == m.h
    lm = lshape_mesh(16)
    r2 = rm.perturb(rm.Mesh(lm.vertices, lm.elements, lm.labels), amplitude=0.2, seed=0)
    assert np.array_equal(r2.vertices, perturb(lm, amplitude=0.2, seed=0).vertices)


def test_adjacency_and_ansatz_match_reference(reference):
    import nlfem.mesh as rm
    from nlfem import assembly as ra
    m = perturb(grid_mesh(9, -0.1, 1.1), amplitude=0.2, seed=1)
    rmesh = rm.Mesh(m.vertices, m.elements, m.labels)
    ga, gb = rm.build_adjacency_graph(rmesh), build_adjacency_graph(m)
    assert np.array_equal(ga.ptr, gb.ptr) and np.array_equal(ga.idx, gb.idx)
    for kind in ("cg", "dg"):
        for n in (1, 2):
            a, b = ra.build_ansatz(rmesh, kind, n), build_ansatz(m, kind, n)
            assert np.array_equal(a.dof_map, b.dof_map) and a.dof_count == b.dof_count
            assert np.array_equal(a.free_mask, b.free_mask)


def test_mesh_validation():
    V = np.array([[0, 0], [1, 0], [0, 1.0]])
    with pytest.raises(ConfigurationError):
        Mesh(V, [[0, 2, 1]], [1])  # clockwise
    with pytest.raises(ConfigurationError):
        Mesh(V, [[0, 1, 1]], [1])
    with pytest.raises(ConfigurationError):
        Mesh(V, [[0, 1, 2]], [7])
    m = Mesh(V, [[0, 1, 2]], [int(Label.DOMAIN)])
    assert abs(m.h - math.sqrt(2.0)) < 1e-15


def test_marshal_validation_matches_reference_errors():
    m = grid_mesh(6, 0.0, 1.0)
    adj = build_adjacency_graph(m)
    ans = build_ansatz(m)
    k = fractional_kernel(0.4, 0.3)
    with pytest.raises(ConfigurationError, match="output component"):
        marshal(m, adj, peridynamic_kernel(0.3), ans)
    with pytest.raises(ConfigurationError, match="rows must be"):
        marshal(m, adj, k, ans, rows="some")
    with pytest.raises(ConfigurationError, match="traversal must be"):
        marshal(m, adj, k, ans, traversal="dfs")
    with pytest.raises(ConfigurationError, match="n_threads"):
        marshal(m, adj, k, ans, n_threads=0)
    with pytest.raises(ConfigurationError, match="continuous ansatz"):
        marshal(m, adj, fractional_kernel(0.7, 0.3), build_ansatz(m, "dg"))
    inp = marshal(m, adj, k, ans, QuadratureConfig())
    assert inp.path_touch == 2 and inp.kernel_id == 0
    assert inp.rskip2 == (1e-13 * m.h) ** 2 and inp.drop2 == 2e-14 * m.h * m.h


def test_c_abi_exports_every_declared_symbol():
    """libnlg.so loads (no GPU needed) and exports every function in include/nlg.h."""
    from paper_2207_03921_b200 import _native
    from paper_2207_03921_b200.build import build
    build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    decl = open(os.path.join(ROOT, "include", "nlg.h")).read()
    names = set(re.findall(r"\b(nlg_[a-z0-9_]+)\(", decl))
    assert names, "no declarations parsed"
    for n in sorted(names):
        assert hasattr(lib, n), f"{n} declared in include/nlg.h but not exported"
    assert set(_native.SIGNATURES) <= names
    assert lib.nlg_abi_version() == 5


def test_label_scaled_kernel_boundary():
    """Label-dependent kernels: a symmetric table over the element labels on a
    built-in base; the host value is table[lx][ly] * base (what a reference
    callable computes, kernels.py:21-35); a nonsymmetric table is refused."""
    from paper_2207_03921_b200 import Label, label_scaled_kernel
    m = generate_structured_mesh(1.0, 0.25, 4)
    adj = build_adjacency_graph(m)
    ans = build_ansatz(m, "cg", 1)
    base = fractional_kernel(0.4, 0.25)
    k = label_scaled_kernel(base, [[1.0, 0.5], [0.5, 2.0]])
    x, y = np.array([0.1, 0.2]), np.array([0.3, 0.25])
    assert k.value(x, y, Label.DOMAIN, Label.DIRICHLET)[0, 0] == 0.5 * base.value(x, y)[0, 0]
    assert k.value(x, y, Label.DIRICHLET, Label.DIRICHLET)[0, 0] == 2.0 * base.value(x, y)[0, 0]
    inp = marshal(m, adj, k, ans)
    assert inp.kernel_id == 0 and inp.label_scale == (0.0, 0.0, 0.0, 0.0, 1.0, 0.5, 0.0, 0.5, 2.0)
    assert marshal(m, adj, base, ans).label_scale == ()
    with pytest.raises(ConfigurationError, match="symmetric"):
        label_scaled_kernel(base, [[1.0, 0.5], [0.25, 2.0]])
    with pytest.raises(ConfigurationError, match="2 x 2"):
        label_scaled_kernel(base, [1.0, 2.0])


def test_pinned_sink_falls_back_to_pageable_memory(monkeypatch):
    """Without page-locked memory the host CSR block is ordinary numpy memory
    (the library's copies still land there); the arrays are views of it."""
    from paper_2207_03921_b200 import _native
    monkeypatch.setattr(_native.PINNED, "take", lambda nbytes: (None, 0))
    sink = _native.PinnedSink()
    first = sink._alloc(None, 4096, 5)
    addr = sink._alloc(None, 1000, 5)   # the library asked twice: the first block is dropped
    assert first and addr and first != addr
    out = _native.HostCsr()
    out.arena, out.nnz, out.off_data, out.off_indices, out.off_indptr = addr, 10, 0, 80, 128
    ip, ix, dv = sink.arrays(out, 4)
    assert (ip.dtype, ix.dtype, dv.dtype) == (np.int64, np.int32, np.float64)
    assert (ip.shape, ix.shape, dv.shape) == ((5,), (10,), (10,))
    assert dv.ctypes.data == addr and ix.ctypes.data == addr + 80 and ip.ctypes.data == addr + 128
    assert sink.blocks == []
