"""Per-step timing diagnostics for the bench workload (event time vs library total)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2207_03921_b200 import configs
from paper_2207_03921_b200.assembly import DevicePlan
from paper_2207_03921_b200.problem import marshal
cfg = configs.build(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
inp = marshal(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad)
plan = DevicePlan(inp, on_device=True)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
import gc
gc.disable()
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    flush.fill_(float(i))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    print(f'[py  {time.monotonic()*1e3:10.3f}] call', file=sys.stderr, flush=True)
    a.record()
    _, _, _, st = plan.assemble(out_on_host=False, reuse_output=True)
    print(f'[py  {time.monotonic()*1e3:10.3f}] returned', file=sys.stderr, flush=True)
    b.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"step {i}: event {a.elapsed_time(b):8.2f} ms  wall {1e3*(t1-t0):8.2f} ms  lib_total {st['ms_total']:8.2f}  "
          f"phases {st['ms_candidates']+st['ms_full']+st['ms_partial']+st['ms_singular']+st['ms_merge']:7.2f}  "
          f"mem {torch.cuda.memory_reserved()/1e9:.1f} GB", flush=True)
