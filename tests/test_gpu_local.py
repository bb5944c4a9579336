"""Per-pair parity: the device's local_contribution (nlg_local_blocks) against
the reference's own local_contribution (assembly.py:327-448) on sampled
ordered pairs -- identical, edge- and vertex-touching (tensor rules on the
regularizing path), inside, near the ball's rim and far -- of seven
fixtures (tests/golden/local_*.npz, made by make_local.py from the
reference), and the reference's cross-check that the blocks of all ordered
pairs sum to the assembled matrix (<= 1.4e-15 there).

Bar: identical rows / columns, block within 1e-10 relative (Frobenius) per pair.
"""

import glob
import os

import numpy as np
import pytest
from scipy import sparse

from golden_io import Case, rel_fro

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
LOCAL = sorted(os.path.basename(p)[6:-4] for p in glob.glob(os.path.join(GOLDEN, "local_*.npz")))


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _plan(c):
    from paper_2207_03921_b200.assembly import DevicePlan
    from paper_2207_03921_b200.problem import marshal
    return DevicePlan(marshal(*c.args(), rows=c.rows))


@pytest.mark.parametrize("name", LOCAL)
def test_local_blocks_match_reference(name):
    z = np.load(os.path.join(GOLDEN, f"local_{name}.npz"))
    c = Case(name)
    plan = _plan(c)
    try:
        got = plan.local_blocks(z["pairs"])
    finally:
        plan.close()
    for i, (k, l) in enumerate(z["pairs"]):
        d = int(z["dims"][i])
        ref, g = z["blocks"][i][:d, :d], got[i]
        assert g.block.shape == (d, d), (k, l)
        assert np.array_equal(g.rows, z["rows"][i][:d]), (k, l, g.rows, z["rows"][i][:d])
        nr = np.linalg.norm(ref)
        err = np.linalg.norm(g.block - ref)
        assert err <= 1e-10 * nr or (nr == 0.0 and err == 0.0), f"{name} pair ({k}, {l}): rel {err / max(nr, 1e-300):.2e}"


def test_local_contribution_api_and_errors():
    from paper_2207_03921_b200 import ConfigurationError, local_contribution
    c = Case("frac_s04_approx_pert")
    z = np.load(os.path.join(GOLDEN, "local_frac_s04_approx_pert.npz"))
    k, l = (int(x) for x in z["pairs"][3])
    ls = local_contribution(k, l, c.kernel, c.ansatz, c.quad, c.mesh)
    d = int(z["dims"][3])
    assert np.array_equal(ls.rows, z["rows"][3][:d]) and np.array_equal(ls.cols, ls.rows)
    assert np.linalg.norm(ls.block - z["blocks"][3][:d, :d]) <= 1e-10 * np.linalg.norm(z["blocks"][3][:d, :d])
    with pytest.raises(ConfigurationError, match="out of range"):
        local_contribution(0, c.mesh.n_elements, c.kernel, c.ansatz, c.quad, c.mesh)


@pytest.mark.parametrize("name", ["frac_s04_approx_pert", "peri_approx_transform", "lshape16_affine",
                                  "frac_s04_nocaps_dg"])
def test_sum_of_local_blocks_is_the_assembled_matrix(name):
    """Scatter the blocks of every ordered pair (outer root k, active l) and
    compare with bfs_assemble (the reference's own cross-check)."""
    from paper_2207_03921_b200 import bfs_assemble
    c = Case(name)
    from paper_2207_03921_b200.problem import marshal
    inp = marshal(*c.args(), rows=c.rows)
    roots = np.flatnonzero(inp.outer_mask)
    act = np.flatnonzero(c.mesh.labels != 0)
    pairs = np.stack(np.meshgrid(roots, act, indexing="ij"), axis=-1).reshape(-1, 2)
    plan = _plan(c)
    try:
        blocks = plan.local_blocks(pairs)
    finally:
        plan.close()
    J = c.ansatz.dof_count
    r = np.concatenate([np.repeat(b.rows, b.rows.size) for b in blocks])
    q = np.concatenate([np.tile(b.cols, b.cols.size) for b in blocks])
    v = np.concatenate([b.block.ravel() for b in blocks])
    S = sparse.csr_matrix((v, (r, q)), shape=(J, J))
    A = bfs_assemble(*c.args(), rows=c.rows).matrix
    assert rel_fro(S, A) <= 1e-12
