import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/quick.json"))
print(f"value {d['value']:.4g} EPI/s  ms/step {d['ms_per_step']:.2f}")
print({k: round(v, 2) for k, v in d["roofline"]["phase_ms"].items()})
r = d["roofline"]
print(f"dominant {r['kernel']} {r['achieved']:.2f}/{r['peak']:.1f} TF/s frac {r['frac']:.3f}; all-integration {r['all_integration']['tflops']:.2f} TF/s")
if d.get("e2e"): print("e2e", d["e2e"])
if d.get("cpu_baseline"): print("cpu", d["cpu_baseline"])
print("clocks", d.get("clocks"))
