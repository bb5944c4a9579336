"""Break down the public bfs_assemble (host in / host out) path."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2207_03921_b200 import configs, bfs_assemble
from paper_2207_03921_b200.assembly import DevicePlan, csr_from_parts
from paper_2207_03921_b200.problem import marshal
cfg = configs.build(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
adj = cfg.adjacency
for i in range(3):
    t = [time.perf_counter()]
    inp = marshal(cfg.mesh, adj, cfg.kernel, cfg.ansatz, cfg.quad); t.append(time.perf_counter())
    plan = DevicePlan(inp); t.append(time.perf_counter())
    ip, ix, dv, st = plan.assemble(out_on_host=True); t.append(time.perf_counter())
    plan.close(); t.append(time.perf_counter())
    ta = time.perf_counter(); _ = ip.sum(); _ = ix.max(); _ = dv.sum(); tb = time.perf_counter()
    m = csr_from_parts(ip, ix, dv, inp.n_dofs, inp.n_dofs, canonical=True); t.append(time.perf_counter())
    print(f"  touch {1e3*(tb-ta):.1f} ms; dtypes {ip.dtype} {ix.dtype} {dv.dtype} contiguous {ix.flags.c_contiguous}")
    from scipy import sparse
    for name, f in [("raw", lambda: sparse.csr_matrix((dv, ix, ip), shape=(inp.n_dofs,)*2)),
                    ("i32ptr", lambda: sparse.csr_matrix((dv, ix, ip.astype(np.int32)), shape=(inp.n_dofs,)*2)),
                    ("copies", lambda: sparse.csr_matrix((dv.copy(), ix.copy(), ip.astype(np.int32)), shape=(inp.n_dofs,)*2))]:
        tc = time.perf_counter(); f(); print(f"  scipy {name}: {1e3*(time.perf_counter()-tc):.1f} ms")
    d = np.diff(np.array(t)) * 1e3
    print(f"marshal {d[0]:.1f}  plan {d[1]:.1f}  assemble {d[2]:.1f} (lib {st['ms_total']:.1f})  close {d[3]:.1f}  csr {d[4]:.1f}")
t0 = time.perf_counter(); s = bfs_assemble(cfg.mesh, adj, cfg.kernel, cfg.ansatz, cfg.quad); print("bfs_assemble", (time.perf_counter()-t0)*1e3)
