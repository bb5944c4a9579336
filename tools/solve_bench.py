"""Config-2 end to end on the device: assemble, load vector, Dirichlet split,
CG to 1e-10.  Prints one JSON line."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2207_03921_b200 import assemble_load, bfs_assemble, configs
from paper_2207_03921_b200.solve import cg_device, solve_dirichlet

cfg = configs.build(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
sysm = bfs_assemble(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad)
b = assemble_load(cfg.mesh, cfg.ansatz, cfg.f, cfg.quad)
a_ff, _ = sysm.split()
free = np.flatnonzero(sysm.free_mask)
cg_device(a_ff, b[free], rtol=1e-10)  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
u, info = solve_dirichlet(sysm, b, rtol=1e-10)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
r = sysm.matrix @ u - b
print(json.dumps({"config": cfg.name, "n_free": int(free.size), "nnz_free": int(a_ff.nnz), **info,
                  "solve_ms_incl_transfers": dt * 1e3,
                  "ms_per_iteration": dt * 1e3 / max(info["iterations"], 1),
                  "spmv_bytes_per_iteration": int(a_ff.nnz * 12 + free.size * 24),
                  "free_residual_rel": float(np.linalg.norm(r[sysm.free_mask]) / np.linalg.norm(b[sysm.free_mask]))}))
