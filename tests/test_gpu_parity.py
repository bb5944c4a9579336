"""GPU parity: libnlg.so through the public bfs_assemble / assemble_load
against the reference (golden fixtures it produced) and the CPU oracle.

Bar (BASELINE.json north_star): identical sparsity pattern, bit for bit;
values within 1e-10 relative Frobenius; load vector within 1e-10 relative
2-norm.
"""

import math

import numpy as np
import pytest
from scipy import sparse

from golden_io import Case, names, rel_fro, same_pattern
from oracle import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_03921_b200 import _native
    _native.load_library()
    oracle.build()


def _gpu_matrix(c, **kw):
    from paper_2207_03921_b200 import bfs_assemble
    return bfs_assemble(*c.args(), rows=c.rows, **kw)


@pytest.mark.parametrize("name", names())
def test_golden_pattern_and_values(name):
    c = Case(name)
    st = {}
    sysm = _gpu_matrix(c, stats=st)
    A = sysm.matrix
    assert A.shape == c.matrix.shape
    assert same_pattern(A, c.matrix), f"{name}: pattern differs (nnz {A.nnz} vs {c.matrix.nnz})"
    err = rel_fro(A, c.matrix)
    assert err <= TOL, f"{name}: rel Frobenius error {err:.3e}"
    assert np.array_equal(sysm.free_mask, c.free_mask)


@pytest.mark.parametrize("name", names())
def test_golden_load(name):
    from paper_2207_03921_b200 import assemble_load
    c = Case(name)
    b = assemble_load(c.mesh, c.ansatz, c.f, c.quad)
    assert np.linalg.norm(b - c.b) <= TOL * np.linalg.norm(c.b)


def test_load_constant_on_device_partition_of_unity():
    from paper_2207_03921_b200 import assemble_load
    c = Case("cfg1_approxcaps")
    b = assemble_load(c.mesh, c.ansatz, 1.0)
    assert np.linalg.norm(b - c.b) <= TOL * np.linalg.norm(c.b)
    assert abs(b.sum() - 1.44) <= 1e-12  # area of [-0.1, 1.1]^2


@pytest.mark.parametrize("name", ["frac_s04_approx_pert", "cfg1_approxcaps", "lshape16_affine", "peri_nocaps_avoid",
                                  "peri_approx_transform", "const_inf_pert", "frac_s04_nocaps_dg"])
def test_deterministic_and_row_split_invariant(name):
    """Run-to-run bitwise determinism, and the reference's thread-count
    invariance carried over to the GPU row split: owner-computed
    row blocks -- what each GPU of a multi-GPU run assembles -- and small
    memory-budget batches concatenate into the full matrix BIT FOR BIT.
    (Pair records are integrated in canonical orientation, the merge sums in
    exact fixed point, and each row's fixed-point scale comes from its own
    elements' bounds.)"""
    from paper_2207_03921_b200 import bfs_assemble
    c = Case(name)
    a = bfs_assemble(*c.args(), rows=c.rows).matrix
    b = bfs_assemble(*c.args(), rows=c.rows).matrix
    assert np.array_equal(a.data, b.data)  # run-to-run bitwise
    J = c.ansatz.dof_count
    nc = c.ansatz.n
    for cuts in ([0, J // 7, J // 3, (2 * J) // 3, J], [0, J // 2, J]):
        cuts = [x // nc * nc for x in cuts[:-1]] + [J]
        blocks = [bfs_assemble(*c.args(), rows=c.rows, row_range=(lo, hi)).matrix for lo, hi in zip(cuts[:-1], cuts[1:])]
        whole = sparse.vstack(blocks).tocsr()
        assert np.array_equal(whole.indptr, a.indptr) and np.array_equal(whole.indices, a.indices)
        assert np.array_equal(whole.data, a.data), f"{name}: row split {cuts} changes values " \
            f"(max rel {np.max(np.abs(whole.data - a.data)) / np.max(np.abs(a.data)):.2e})"
    st = {}
    small = bfs_assemble(*c.args(), rows=c.rows, mem_budget=1 << 20, stats=st).matrix
    assert st["n_batches"] > 1
    assert np.array_equal(small.indices, a.indices) and np.array_equal(small.data, a.data)


def test_small_memory_budget_batches():
    from paper_2207_03921_b200 import bfs_assemble
    c = Case("peri_nocaps_avoid")
    st = {}
    a = bfs_assemble(*c.args()).matrix
    b = bfs_assemble(*c.args(), mem_budget=4 << 20, stats=st).matrix
    assert st["n_batches"] > 1
    assert same_pattern(a, b) and np.array_equal(a.data, b.data)  # batching never changes a value
    assert same_pattern(b, c.matrix) and rel_fro(b, c.matrix) <= TOL


@pytest.mark.parametrize("traversal", ["bfs", "brute"])
def test_nonfinite_contribution_raises_numerical_error_naming_the_reference_pair(traversal):
    """A nonfinite kernel scale: NumericalError naming the pair the
    reference names (assembly.py:285-288) -- the first failing visit of the
    smallest failing root, in the traversal's visiting order."""
    from paper_2207_03921_b200 import NumericalError, bfs_assemble, constant_kernel
    c = Case("cfg1_nocaps")
    k = constant_kernel(0.1, "nocaps", scale=float("nan"))
    ref, r = oracle.assemble(c.mesh, c.adjacency, k, c.ansatz, rows="domain", traversal=traversal)
    assert r["err"] == 1
    with pytest.raises(NumericalError, match=rf"element pair \({r['ek']}, {r['el']}\)$"):
        bfs_assemble(c.mesh, c.adjacency, k, c.ansatz, rows="domain", traversal=traversal)


def test_callable_kernel_rejected():
    from paper_2207_03921_b200 import ConfigurationError, KernelSpec, bfs_assemble
    c = Case("cfg1_nocaps")
    k = KernelSpec(delta=0.1, s=-1.0, n=1, symmetric=True, ball="nocaps", value=lambda *a: [[1.0]])
    with pytest.raises(ConfigurationError):
        bfs_assemble(c.mesh, c.adjacency, k, c.ansatz)


def _cfg(n):
    from paper_2207_03921_b200 import configs
    return configs.build(n)


@pytest.mark.slow
def test_cfg2_full_matches_survey_and_oracle_band():
    """Config 2 (N=128, fractional s=0.4, approxcaps, singular path): full GPU
    matrix vs the survey's recorded reference numbers and vs the oracle on a
    band of complete rows."""
    from paper_2207_03921_b200 import bfs_assemble
    cfg = _cfg(2)
    st = {}
    A = bfs_assemble(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, stats=st).matrix
    assert A.nnz == 7336929  # SURVEY.md 8c, reference measured
    assert abs(np.linalg.norm(A.data) - 38.40221826904719) <= 1e-10 * 38.4
    assert st["epi"] == 28118976  # = the oracle's count of the reference's visits (test_gpu_bench_paths)
    # oracle over cell rows [40, 48): complete vertex lines [42, 47]
    N = 128
    lo, hi = oracle.band_rows(N, 40, 48, path_touch=2)
    from paper_2207_03921_b200.problem import marshal
    inp = marshal(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz)
    op = oracle.OracleProblem(inp, cfg.adjacency)
    starts = np.arange(2 * N * 40, 2 * N * 48, 64)
    ref = op.run(starts=starts, ends=np.minimum(starts + 64, 2 * N * 48))
    R = sparse.csr_matrix((ref["data"], ref["indices"], ref["indptr"]), shape=A.shape)[lo:hi]
    G = A[lo:hi]
    assert same_pattern(G, R)
    assert rel_fro(G, R) <= TOL


@pytest.mark.slow
def test_cfg1_properties():
    from paper_2207_03921_b200 import bfs_assemble
    cfg = _cfg(1)
    A = bfs_assemble(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz).matrix
    asym = abs(A - A.T).max()
    assert asym <= 1e-12 * abs(A).max()  # SPEC.md:402 symmetry


def test_neumann_null_space():
    """Pure Neumann constant-kernel assembly: ||A 1||_inf <= 1e-12 ||A||_max J."""
    from paper_2207_03921_b200 import (Mesh, bfs_assemble, build_adjacency_graph, build_ansatz,
                                       constant_kernel, grid_mesh, perturb)
    m = perturb(grid_mesh(24, 0.0, 1.0), amplitude=0.2, seed=5)
    m = Mesh(m.vertices, m.elements, np.ones(m.n_elements, dtype=np.int64))
    ans = build_ansatz(m, "cg", 1)
    A = bfs_assemble(m, build_adjacency_graph(m), constant_kernel(0.15, "approxcaps"), ans).matrix
    assert np.abs(A @ np.ones(A.shape[0])).max() <= 1e-12 * abs(A).max() * A.shape[0]


def test_nonsymmetric_column_sums_vanish():
    """For the nonsymmetric affine kernel only 1^T A vanishes."""
    c = Case("lshape16_affine")
    A = _gpu_matrix(c).matrix
    assert np.abs(np.ones(A.shape[0]) @ A).max() <= 1e-12 * abs(A).max() * A.shape[0]
    assert math.isfinite(A.data.sum())
