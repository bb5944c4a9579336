"""Device-resident assembly time vs memory budget (fewer row batches = fewer pairs integrated twice at the cuts)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2207_03921_b200 import configs
from paper_2207_03921_b200.assembly import DevicePlan
from paper_2207_03921_b200.problem import marshal
cfg = configs.build(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
inp = marshal(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad)
tot = torch.cuda.mem_get_info(0)[1]
plan = DevicePlan(inp, on_device=True)
for frac in [float(x) for x in sys.argv[2:]] or [0.6, 0.75, 0.85]:
    for i in range(3):
        try:
            _, _, _, st = plan.assemble(out_on_host=False, reuse_output=True, mem_budget=int(frac * tot))
        except Exception as e:  # noqa: BLE001
            print(f"budget {frac}: {type(e).__name__}: {e}")
            break
        torch.cuda.synchronize()
        free = torch.cuda.mem_get_info(0)[0] / 1e9
        print(f"budget {frac:.2f} call {i}: {st['ms_total']:.1f} ms, batches {st['n_batches']} replans {st['n_replans']}, "
              f"cand {st['ms_candidates']:.1f} partial {st['ms_partial']:.1f} merge {st['ms_merge']:.1f}, free now {free:.1f} GB", flush=True)
