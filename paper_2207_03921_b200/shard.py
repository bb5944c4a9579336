"""Owner-computes row sharding across the GPUs of one node.

Each rank owns a contiguous, vertex-aligned range of CSR rows and assembles
exactly those rows (``nlg_assemble(row_lo, row_hi)``: every outer element
whose block reaches an owned row is evaluated, only owned rows are emitted),
so the row blocks are disjoint and concatenate into the full matrix with no
reduction collective on the data path.  The only communication is the
optional final gather of the row blocks (``torch.distributed``: NCCL between
GPUs, gloo in the CPU tests).

The reference has no distributed path (threads over 64-root spans,
assembly.py:245-283); this module replaces the span partition.
"""

import numpy as np
from scipy import sparse

from .mesh import Label


def vertex_work(mesh, ansatz):
    """Per-dof-base work estimate: active elements incident to each base dof.

    A row's cost is the candidate pairs of the outer elements that reach it,
    which on a quasi-uniform mesh is proportional to its incident elements.
    """
    act = mesh.labels != Label.INACTIVE
    nbase = ansatz.dof_count // ansatz.n
    return np.bincount(ansatz.dof_map[act].ravel(), minlength=nbase).astype(np.float64)


def row_partition(n_dofs, nc, world_size, weights=None):
    """Cut points [0 = c_0 <= ... <= c_W = n_dofs] on dof-base boundaries,
    balancing ``weights`` (per dof base) when given, else the row count."""
    nbase = n_dofs // nc
    if weights is None:
        cuts = [nc * (nbase * r // world_size) for r in range(world_size + 1)]
    else:
        cum = np.concatenate([[0.0], np.cumsum(np.asarray(weights, dtype=np.float64))])
        targets = cum[-1] * np.arange(world_size + 1) / world_size
        cuts = [nc * int(np.searchsorted(cum, t, side="left")) for t in targets]
    cuts[0], cuts[-1] = 0, n_dofs
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return cuts


def my_rows(n_dofs, nc, rank, world_size, weights=None):
    cuts = row_partition(n_dofs, nc, world_size, weights)
    return cuts[rank], cuts[rank + 1]


def gather_blocks(block, n_cols, group=None, dst=0, device=None):
    """Gather CSR row blocks (rank order) into one matrix on ``dst``.

    ``block`` is a scipy CSR matrix of this rank's rows.  Sizes are exchanged
    first, then padded tensors are gathered (NCCL needs equal shapes).
    Returns the stacked matrix on ``dst`` and None elsewhere.
    """
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    b = block.tocsr()
    sizes = torch.tensor([b.shape[0], b.nnz], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(ws)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [tuple(int(v) for v in t.cpu()) for t in all_sizes]
    max_rows = max(r for r, _ in all_sizes)
    max_nnz = max(n for _, n in all_sizes)

    def padded(arr, n, dtype):
        t = torch.zeros(max(n, 1), dtype=dtype, device=dev)
        if arr.size:
            t[:arr.size] = torch.as_tensor(np.ascontiguousarray(arr), dtype=dtype).to(dev)
        return t

    parts = {}
    for name, arr, n, dt in (("indptr", b.indptr, max_rows + 1, torch.int64),
                             ("indices", b.indices, max_nnz, torch.int64),
                             ("data", b.data, max_nnz, torch.float64)):
        mine = padded(arr, n, dt)
        bufs = [torch.zeros_like(mine) for _ in range(ws)]
        dist.all_gather(bufs, mine, group=group)
        parts[name] = bufs
    if rank != dst:
        return None
    blocks = []
    for r, (nr, nz) in enumerate(all_sizes):
        ip = parts["indptr"][r][:nr + 1].cpu().numpy()
        blocks.append(sparse.csr_matrix((parts["data"][r][:nz].cpu().numpy(),
                                         parts["indices"][r][:nz].cpu().numpy(), ip),
                                        shape=(nr, n_cols)))
    return sparse.vstack(blocks).tocsr()


def assemble_sharded(mesh, adjacency, kernel, ansatz, quad=None, rows="all", group=None,
                     device=None, gather=True, block_fn=None, balance=True):
    """Assemble this rank's row block and (optionally) gather the full matrix.

    ``block_fn(lo, hi)`` computes the CSR rows [lo, hi); it defaults to the
    GPU ``bfs_assemble(..., row_range=(lo, hi))`` on ``device``.
    Returns (row_range, block, full_or_None).
    """
    import torch.distributed as dist
    ws = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    weights = vertex_work(mesh, ansatz) if balance else None
    lo, hi = my_rows(ansatz.dof_count, ansatz.n, rank, ws, weights)
    if block_fn is None:
        from .assembly import bfs_assemble

        def block_fn(a, b):
            return bfs_assemble(mesh, adjacency, kernel, ansatz, quad, rows=rows,
                                device=0 if device is None else device, row_range=(a, b)).matrix
    block = block_fn(lo, hi)
    full = None
    if gather and ws > 1:
        full = gather_blocks(block, ansatz.dof_count, group=group,
                             device=None if device is None or not _is_nccl(group) else f"cuda:{device}")
    elif gather:
        full = block
    return (lo, hi), block, full


def _is_nccl(group):
    import torch.distributed as dist
    return dist.get_backend(group) == "nccl"
