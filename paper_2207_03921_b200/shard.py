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


def owner_roots(mesh, ansatz, lo, hi, outer_mask, path_touch):
    """Outer elements a rank owning CSR rows [lo, hi) evaluates (host mirror
    of the device's k_mark_a / k_mark_vertices / k_mark_roots): the elements
    with a dof row in the range, plus -- on the regularizing path, where a
    touching pair is integrated by its smaller root only (_engine.py:233) --
    every outer element touching one of them."""
    nc = ansatz.n
    d = np.asarray(ansatz.dof_map, dtype=np.int64)
    need = ((nc * d + nc - 1 >= lo) & (nc * d < hi)).any(axis=1)
    outer = np.asarray(outer_mask) != 0
    roots = outer & need
    if path_touch == 2:
        vmark = np.zeros(mesh.n_vertices, dtype=bool)
        vmark[mesh.elements[need].ravel()] = True
        roots |= outer & vmark[mesh.elements].any(axis=1)
    return np.flatnonzero(roots)


def row_weights(plan, mesh=None, ansatz=None):
    """EPI-balanced per-dof-base weights (split by EPI prefix
    sums): the device's per-root visit counts summed onto the root's dofs
    (``DevicePlan.row_work``).  Boundary strips are cheaper than interior
    ones (up to ~7% at config 4), which incident-element counts miss.
    Without a plan, falls back to :func:`vertex_work`."""
    if plan is None:
        return vertex_work(mesh, ansatz)
    return plan.row_work().astype(np.float64)


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


def _send_array(arr, dst, dev, chunk, group):
    import torch
    import torch.distributed as dist
    flat = np.ascontiguousarray(arr).reshape(-1)
    for i in range(0, flat.size, chunk):
        t = torch.from_numpy(flat[i:i + chunk]).to(dev)
        dist.send(t, dst, group=group)


def _recv_array(n, dtype, src, dev, chunk, group):
    import torch
    import torch.distributed as dist
    out = np.empty(n, dtype=dtype)
    tdt = {np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
           np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
    buf = torch.empty(min(max(n, 1), chunk), dtype=tdt, device=dev)
    for i in range(0, n, chunk):
        m = min(chunk, n - i)
        view = buf[:m]
        dist.recv(view, src, group=group)
        out[i:i + m] = view.cpu().numpy()
    return out


def gather_blocks(block, n_cols, group=None, dst=0, device=None, chunk_bytes=1 << 30):
    """Gather CSR row blocks (rank order) into one host matrix on ``dst``.

    Point-to-point: every rank sends its own block's arrays (exact sizes,
    no padding) to ``dst`` in chunks of at most ``chunk_bytes``; ``dst``
    receives them into one reusable staging tensor and lands them in host
    memory, so no rank ever holds more than its own block plus one chunk on
    the device (config 4: ~33 GB per rank, ~266 GB in total on the host of
    ``dst``).  ``device``: the NCCL device of this rank (None: CPU / gloo).
    Returns the stacked scipy CSR on ``dst`` and None elsewhere.
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
    gdst = dist.get_global_rank(group, dst) if group is not None else dst
    ind_dt = np.int64 if max(n for _, n in all_sizes) >= 2 ** 31 or n_cols >= 2 ** 31 else np.int32
    arrays = lambda m: (np.asarray(m.indptr, dtype=np.int64), np.asarray(m.indices, dtype=ind_dt),  # noqa: E731
                        np.asarray(m.data, dtype=np.float64))
    if rank != dst:
        for arr in arrays(b):
            _send_array(arr, gdst, dev, max(1, chunk_bytes // arr.itemsize), group)
        return None
    blocks = []
    for r, (nr, nz) in enumerate(all_sizes):
        if r == dst:
            ip, ix, dv = arrays(b)
        else:
            src = dist.get_global_rank(group, r) if group is not None else r
            ip = _recv_array(nr + 1, np.int64, src, dev, chunk_bytes // 8, group)
            ix = _recv_array(nz, ind_dt, src, dev, chunk_bytes // np.dtype(ind_dt).itemsize, group)
            dv = _recv_array(nz, np.float64, src, dev, chunk_bytes // 8, group)
        blocks.append(sparse.csr_matrix((dv, ix, ip), shape=(nr, n_cols)))
    return sparse.vstack(blocks, format="csr")


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
    if block_fn is None:
        from .assembly import DevicePlan, bfs_assemble
        from .problem import marshal
        weights = None
        if balance:  # EPI prefix sums from the device count pass (same on every rank)
            plan = DevicePlan(marshal(mesh, adjacency, kernel, ansatz, quad, rows=rows),
                              device=0 if device is None else device)
            try:
                weights = row_weights(plan)
            finally:
                plan.close()
    else:
        weights = vertex_work(mesh, ansatz) if balance else None
    lo, hi = my_rows(ansatz.dof_count, ansatz.n, rank, ws, weights)
    if block_fn is None:

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
