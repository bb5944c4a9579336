"""Phase times of the host-output path (DevicePlan.assemble(out_on_host=True)) over a few calls."""
import sys, time
sys.path.insert(0, ".")
from paper_2207_03921_b200 import configs
from paper_2207_03921_b200.assembly import DevicePlan
from paper_2207_03921_b200.problem import marshal
cfg = configs.build(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
inp = marshal(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad)
for i in range(4):
    plan = DevicePlan(inp)
    t0 = time.perf_counter()
    ip, ix, dv, st = plan.assemble(out_on_host=True)
    dt = (time.perf_counter() - t0) * 1e3
    plan.close()
    del ip, ix, dv
    print(f"call {i}: {dt:.1f} ms wall, lib {st['ms_total']:.1f}, batches {st['n_batches']} replans {st['n_replans']}, "
          f"cand {st['ms_candidates']:.1f} partial {st['ms_partial']:.1f} merge {st['ms_merge']:.1f} prep {st['ms_prep']:.1f}")
