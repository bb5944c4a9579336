"""Debug: cfg5 (reduced grid) with a small memory budget (many batches)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2207_03921_b200 import configs, bfs_assemble
n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
budget = int(float(sys.argv[2])) if len(sys.argv) > 2 else 0
cfg = configs.build(5, grid_n=n)
st = {}
A = bfs_assemble(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad, mem_budget=budget, stats=st).matrix
print("nnz", A.nnz, "batches", st["n_batches"], "replans", st["n_replans"], "coo", st["coo_entries"], st["coo_reduced"])
