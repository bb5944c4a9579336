"""Multi-rank row sharding on CPU (world_size 2, gloo): the partition is
vertex-aligned and balanced, owner-computed blocks concatenate to the full
matrix, and the gather over torch.distributed reassembles it.  The per-rank
block compute here is the CPU oracle (test infrastructure); on GPUs it is
bfs_assemble(row_range=...), covered by tests/test_gpu_parity.py."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_io import Case
from paper_2207_03921_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_properties():
    c = Case("cfg1_approxcaps")
    w = shard.vertex_work(c.mesh, c.ansatz)
    for ws in (1, 2, 3, 4, 8):
        cuts = shard.row_partition(c.ansatz.dof_count, 1, ws, w)
        assert cuts[0] == 0 and cuts[-1] == c.ansatz.dof_count and len(cuts) == ws + 1
        assert all(a <= b for a, b in zip(cuts, cuts[1:]))
        loads = [w[a:b].sum() for a, b in zip(cuts, cuts[1:])]
        assert max(loads) <= 1.25 * np.mean(loads) + w.max()
    cuts2 = shard.row_partition(450, 2, 4)  # nc = 2: cuts on even rows
    assert all(x % 2 == 0 for x in cuts2)


def _worker(rank, ws, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from golden_io import Case as C2
        from oracle import oracle
        c = C2(name)
        full_ref, _ = oracle.assemble(*c.args(), rows=c.rows)

        def block_fn(lo, hi):
            return full_ref[lo:hi]

        (lo, hi), block, full = shard.assemble_sharded(c.mesh, c.adjacency, c.kernel, c.ansatz, c.quad,
                                                       rows=c.rows, block_fn=block_fn)
        if rank == 0:
            same = (np.array_equal(full.indptr, c.matrix.indptr) and np.array_equal(full.indices, c.matrix.indices)
                    and np.array_equal(full.data, c.matrix.data))
            q.put((lo, hi, bool(same)))
        else:
            q.put((lo, hi, full is None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg1_nocaps", "peri_nocaps_avoid"])
def test_two_rank_gloo_gather_reassembles(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert res[0][0] == 0 and res[0][1] == res[1][0]  # contiguous, disjoint row ranges
    assert all(r[2] for r in res)
