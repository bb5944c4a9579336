"""Stress: rows with more distinct columns than the largest stage-W table
(constant kernel, delta/h ~ 48).  These now run as two column halves in
stage W (no stage-R fallback); the result is compared with NLG_MERGE=sort."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2207_03921_b200 import (bfs_assemble, build_adjacency_graph, build_ansatz, constant_kernel, grid_mesh)
d = 0.3
mesh = grid_mesh(256, -d, 1.0 + d, delta=d)
adj = build_adjacency_graph(mesh)
kern = constant_kernel(d, "approxcaps")
ans = build_ansatz(mesh, "cg", 1)
J = ans.dof_count
rr = (J // 2 - 1500, J // 2 + 1500)
st = {}
t0 = time.time()
a = bfs_assemble(mesh, adj, kern, ans, row_range=rr, stats=st).matrix
print("stage W:", round(time.time() - t0, 2), "s nnz", a.nnz, "max row nnz", np.diff(a.indptr).max(),
      {k: st[k] for k in ("n_batches", "n_replans", "n_row_retries", "n_merge_fallbacks")})
os.environ["NLG_MERGE"] = "sort"
b = bfs_assemble(mesh, adj, kern, ans, row_range=rr).matrix
same = np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
rel = np.linalg.norm((a - b).data) / np.linalg.norm(b.data)
print("pattern equal", same, "rel", rel)
