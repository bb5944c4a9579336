"""GPU: the alternative device paths give the same matrix.

* merge stage W (per-row fixed-point tables) vs the stage R + global sort
  fallback (NLG_MERGE=sort);
* stage W table retries and the fallback itself, forced on small fixtures
  by lowering the table fill limit (NLG_ROW_FILL_DIV);
* analytic full pairs of the constant / affine kernels vs integrating them
  per record (NLG_NO_ANALYTIC);
* the clipped-pair kernel's schedules (NLG_CLIP_WL): bitwise equal.

The switches are read when a plan is created, so each call sets its own
environment.  Same pattern bit for bit; values within 1e-13 relative
Frobenius of each other and within the 1e-10 parity bar of the reference
fixture.
"""

import os

import numpy as np
import pytest

from golden_io import Case, names, rel_fro, same_pattern

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_03921_b200 import _native
    _native.load_library()


def _assemble(c, env=None, **kw):
    from paper_2207_03921_b200 import bfs_assemble
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        return bfs_assemble(*c.args(), rows=c.rows, **kw).matrix
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _agree(a, b, ref):
    assert same_pattern(a, b), f"pattern differs (nnz {a.nnz} vs {b.nnz})"
    assert rel_fro(a, b) <= 1e-13
    assert same_pattern(b, ref) and rel_fro(b, ref) <= TOL


@pytest.mark.parametrize("name", names())
def test_stage_w_matches_stage_r_and_sort(name):
    c = Case(name)
    _agree(_assemble(c), _assemble(c, {"NLG_MERGE": "sort"}), c.matrix)


@pytest.mark.parametrize("name", ["cfg1_approxcaps", "frac_s04_approx_pert", "peri_nocaps_avoid", "lshape16_affine"])
def test_stage_w_retries_and_fallback(name):
    c = Case(name)
    a = _assemble(c)
    st = {}
    # tables overflow early: rows retry in larger tables (nc = 2 tables stop
    # at 2048 slots, so a milder limit keeps the largest one sufficient)
    div = "16" if name.startswith("peri") else "64"
    _agree(a, _assemble(c, {"NLG_ROW_FILL_DIV": div}, stats=st), c.matrix)
    assert st["n_row_retries"] > 0 and st["n_merge_fallbacks"] == 0
    # at 8 columns no table suffices: the batch falls back to stage R + sort
    st = {}
    _agree(a, _assemble(c, {"NLG_ROW_FILL_DIV": "1024"}, stats=st), c.matrix)
    assert st["n_merge_fallbacks"] > 0


@pytest.mark.parametrize("name", [n for n in names() if n.startswith(("cfg1", "const", "lshape16"))])
def test_analytic_full_pairs_match_integrated(name):
    c = Case(name)
    _agree(_assemble(c), _assemble(c, {"NLG_NO_ANALYTIC": "1"}), c.matrix)


@pytest.mark.parametrize("name", ["cfg1_approxcaps", "lshape16_affine", "peri_nocaps_avoid"])
def test_stage_w_column_split_rows(name):
    """Rows too wide for the largest table run as two column halves (below /
    from the row's own dof base): a limit just under the widest rows forces
    it without any fallback.  The peridynamic case runs the nc = 2 split
    kernel (tables keyed by column dof base, 2048 slots at most)."""
    c = Case(name)
    a = _assemble(c, {"NLG_MERGE": "sort"})
    widest = int(np.diff(a.indptr).max())
    if name.startswith("peri"):  # keys are column dof bases: widest / 2 of them per row
        div = str(2048 // max(1, widest // 2 - 2))
    else:
        div = str(8192 // max(1, widest - 4))  # the largest table holds fewer columns than the widest rows
    st = {}
    b = _assemble(c, {"NLG_ROW_FILL_DIV": div}, stats=st)
    assert st["n_merge_fallbacks"] == 0 and st["n_row_retries"] > 0
    _agree(a, b, c.matrix)


@pytest.mark.parametrize("name", [n for n in names() if n.startswith(("cfg1", "const", "lshape16"))])
@pytest.mark.parametrize("variant", ["3", "5", "9", "11", "18"])
def test_clip_ring_schedules_same_bits(name, variant):
    """k_clipped_cfr (clip queue as a ring across rounds, block shapes and
    barriers of NLG_CLIP_WL = 5 / 9 / 11 / 18 / default) computes every item
    as k_clipped_cf (3: no ring) does and folds it by the same shuffles:
    another schedule, the same bits."""
    c = Case(name)
    a = _assemble(c)
    b = _assemble(c, {"NLG_CLIP_WL": variant})
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data, b.data)


def test_stage_w_deterministic_across_table_sizes():
    """Fixed-point sums are exact: the same row summed in a larger table
    (after a retry) gives bitwise the same values."""
    c = Case("cfg1_approxcaps")
    a = _assemble(c)
    b = _assemble(c, {"NLG_ROW_FILL_DIV": "32"})
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data, b.data)


def test_pinned_host_output_pool():
    """Host CSR through nlg_assemble_pinned (views of a pooled page-locked
    block) equals the staged nlg_assemble path bit for bit; a live result is
    never overwritten by a later assembly, and a dropped one is recycled."""
    import gc
    from paper_2207_03921_b200 import _native
    c = Case("lshape16_affine")
    staged = _assemble(c, {"NLG_NO_PINNED_OUTPUT": "1"})
    a1 = _assemble(c)
    snap = (a1.indptr.copy(), a1.indices.copy(), a1.data.copy())
    a2 = _assemble(c)  # a1 still alive: another block
    assert a2.data.ctypes.data != a1.data.ctypes.data
    for m in (a1, a2):
        assert np.array_equal(m.indptr, staged.indptr) and np.array_equal(m.indices, staged.indices)
        assert np.array_equal(m.data, staged.data)
    assert np.array_equal(a1.indptr, snap[0]) and np.array_equal(a1.indices, snap[1]) and np.array_equal(a1.data, snap[2])
    assert same_pattern(a1, c.matrix) and rel_fro(a1, c.matrix) <= TOL
    del a1, a2, m
    gc.collect()
    n0 = _native.PINNED.n_alloc
    a3 = _assemble(c)  # steady state: a pooled block, no new pinning
    assert _native.PINNED.n_alloc == n0
    assert np.array_equal(a3.data, staged.data)
