"""Parity on exactly the paths bench.py times (GPU).

* the EPI numerator of the metric: the device's in-kernel count equals the
  CPU oracle's count of the reference's visits (brute traversal,
  _engine.py:219-225 / :486-490) -- configs 1, 2, 5 reduced and 5 full, and
  config 4's rank-0 row range (EPI home rule: roots whose smallest dof row
  lies in the range);
* config 4's rank-0 range [0, hi) of 8 through ``DevicePlan.assemble`` with
  the default memory budget -- the batched path of ``bench.py --config 4
  --emulate-shard 0/8``: complete rows on both sides of every batch cut
  (where each batch re-evaluates its halo roots) and random rows, against
  the oracle;
* full-size load vectors of configs 2-5 against the oracle's restatement of
  assemble_load (assembly.py:451-481).

Bar: bit-exact pattern, values within 1e-10 relative (north_star).
"""

import numpy as np
import pytest
from scipy import sparse

from golden_io import oracle_rows, rel_fro, same_pattern

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle
    oracle.build()


def _cfg(n, **kw):
    from paper_2207_03921_b200 import configs
    return configs.build(n, **kw)


def _oracle_problem(cfg):
    from oracle import oracle
    from paper_2207_03921_b200.problem import marshal
    inp = marshal(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad)
    return inp, oracle.OracleProblem(inp, cfg.adjacency)


def _device_epi(cfg, lo=0, hi=None):
    from paper_2207_03921_b200.assembly import DevicePlan
    inp, _ = _oracle_problem(cfg)
    plan = DevicePlan(inp, on_device=True)
    try:
        _, _, _, st = plan.assemble(lo, inp.n_dofs if hi is None else hi, out_on_host=False)
    finally:
        plan.close()
    return st["epi"]


@pytest.mark.parametrize("n,kw", [(1, {}), (2, {}), (5, {"grid_n": 48}),
                                  pytest.param(5, {}, marks=pytest.mark.slow)])
def test_epi_equals_oracle_visit_count(n, kw):
    cfg = _cfg(n, **kw)
    _, op = _oracle_problem(cfg)
    ref = int(op.count_visits().sum())
    assert _device_epi(cfg) == ref
    if n == 2 and not kw:
        assert ref == 28118976  # config 2 (2.81e7)


def _rows_dev(indptr, indices, data, rows, J):
    """Host CSR of the given local rows of a device-resident CSR."""
    import torch
    r = torch.as_tensor(np.asarray(rows), dtype=torch.int64, device=indptr.device)
    s, e = indptr[r].cpu().numpy(), indptr[r + 1].cpu().numpy()
    cols, vals, ptr = [], [], [0]
    for a, b in zip(s, e):
        cols.append(indices[int(a):int(b)].cpu().numpy())
        vals.append(data[int(a):int(b)].cpu().numpy())
        ptr.append(ptr[-1] + int(b - a))
    return sparse.csr_matrix((np.concatenate(vals), np.concatenate(cols), np.array(ptr)), shape=(len(rows), J))


@pytest.mark.slow
def test_cfg4_rank0_batched_range_at_batch_cuts():
    from paper_2207_03921_b200 import shard
    from paper_2207_03921_b200.assembly import DevicePlan
    cfg = _cfg(4)
    inp, op = _oracle_problem(cfg)
    J, N = inp.n_dofs, cfg.grid_n
    lo, hi = shard.my_rows(J, 1, 0, 8, shard.vertex_work(cfg.mesh, cfg.ansatz))
    plan = DevicePlan(inp, on_device=True)
    try:
        indptr, indices, data, st = plan.assemble(lo, hi, out_on_host=False)
        batches = plan.last_batches()
        assert len(batches) >= 2, "config 4's rank range is expected to run in several batches"
        assert batches[0][0] == lo and batches[-1][1] == hi
        assert all(a[1] == b[0] for a, b in zip(batches, batches[1:]))
        # EPI of the range: roots whose smallest dof row lies in [lo, hi)
        home = inp.dof_map.min(axis=1)
        mine = np.flatnonzero((home >= lo) & (home < hi))
        k0, k1 = int(mine.min()), int(mine.max()) + 1
        vis = op.count_visits(k0, k1)
        assert st["epi"] == int(vis[mine - k0].sum())
        rng = np.random.default_rng(7)
        verts = set()
        for cut in [b[0] for b in batches[1:]]:
            line = cut // (N + 1)
            for dl in range(-2, 3):
                vline = line + dl
                if 0 <= vline <= N:
                    xs = rng.choice(N + 1, size=6, replace=False)
                    verts.update(int(vline * (N + 1) + x) for x in xs)
            verts.update((cut - 1, cut, cut + 1))
        verts.update(int(v) for v in rng.integers(lo, hi, size=50))
        verts = np.array(sorted(v for v in verts if lo <= v < hi), dtype=np.int64)
        rows, R = oracle_rows(inp, cfg.adjacency, cfg.mesh, verts)
        G = _rows_dev(indptr, indices, data, rows - lo, J)
        assert same_pattern(G, R), "rows at the batch cuts: pattern differs"
        err = rel_fro(G, R)
        assert err <= TOL, f"rows at the batch cuts: rel Frobenius {err:.3e}"
    finally:
        plan.close()


@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_full_size_load_vector(n):
    from oracle import oracle
    from paper_2207_03921_b200 import assemble_load
    cfg = _cfg(n)
    b = assemble_load(cfg.mesh, cfg.ansatz, cfg.f, cfg.quad)
    ref = oracle.assemble_load(cfg.mesh, cfg.ansatz, cfg.f, cfg.quad)
    assert b.shape == ref.shape
    assert np.linalg.norm(b - ref) <= TOL * np.linalg.norm(ref)
    # the constant-f path that never leaves the device
    fconst = (0.0, -1.0) if n == 3 else 1.0
    bc = assemble_load(cfg.mesh, cfg.ansatz, fconst, cfg.quad)
    assert np.linalg.norm(bc - ref) <= TOL * np.linalg.norm(ref)
