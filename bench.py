"""Benchmark: full nonlocal stiffness assembly (fp64) on B200 vs the CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

A step is one complete assembly of BASELINE config C (default 2: N=128,
fractional s=0.4, approxcaps, singular path) from mesh
arrays resident in HBM to the CSR resident in HBM: element bounds, grid
hash, candidate search, pair integration, touching-pair tensor rules, sort
and segmented reduction.  ``value`` = evaluated element-pair integrals
(EPI) / second over the whole job.  ``e2e`` repeats the step
through the public drop-in API ``bfs_assemble`` with host numpy inputs and
a host scipy CSR out (H2D and D2H inside the timed region).

Under torchrun each rank owns a contiguous CSR row range (owner computes;
no collective on the data path) and the time is the max over ranks.

``--impl reference`` times the reference algorithm on the host cores: the
C restatement in oracle/ (bit-identical to the reference's numba engine +
merge; the Python reference itself is not present on the GPU box), on a
bounded band of outer elements of the same config.
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "element-pair integrals/sec (full fp64 stiffness assembly)"
UNIT = "EPI/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


class ClockSampler:
    """SM clocks and throttle reasons sampled (in-process NVML) during the timed region."""

    HW, HW_THERM, SW_THERM, SW_POWER = 0x8, 0x40, 0x20, 0x4  # nvmlClocksEventReason* bits

    def __init__(self, index=0, period=float(os.environ.get("NLG_CLOCK_PERIOD", "0.25"))):
        self.index = index
        self.period = period
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                sm = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
                rs = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.rows.append((sm, rs))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        names = {self.HW: "hw_slowdown", self.HW_THERM: "hw_thermal_slowdown",
                 self.SW_THERM: "sw_thermal_slowdown", self.SW_POWER: "sw_power_cap"}
        reasons = sorted({n for _, rs in self.rows for bit, n in names.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm for sm, _ in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, in-process"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference(cfg, budget_s, threads):
    """The reference algorithm (oracle port, bit-identical) on a bounded band
    of outer elements: returns EPI/s, the sample description and seconds."""
    from oracle import oracle
    from paper_2207_03921_b200.problem import marshal
    inp = marshal(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad)
    op = oracle.OracleProblem(inp, cfg.adjacency)
    K = cfg.mesh.n_elements
    mid = K // 2
    # calibrate on a small band, then size the sample to ~budget_s
    n = 2 * 64 * max(threads, 1)
    t0 = time.perf_counter()
    lo = max(0, mid - n // 2)
    r = op.run(*op.spans(lo, min(K, lo + n)), nthreads=threads)
    dt = time.perf_counter() - t0
    per_root = dt / n
    n2 = int(min(K, max(n, budget_s / max(per_root, 1e-9))))
    n2 = max(64, n2 // 64 * 64)
    lo = max(0, mid - n2 // 2)
    t0 = time.perf_counter()
    r = op.run(*op.spans(lo, min(K, lo + n2)), nthreads=threads)
    dt = time.perf_counter() - t0
    return r["epi"] / dt, f"outer elements [{lo}, {lo + n2}) of {K} (64-root spans, BFS, merge)", dt, r["epi"]


def run_reference(args, cfg, ws, rank):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    from oracle import oracle
    oracle.build()
    vals = []
    # each step a bounded sample; the whole run stays within ~2-3 minutes
    per_step = min(args.ref_seconds, 150.0 / max(1, args.warmup + args.steps))
    for i in range(args.warmup + args.steps):
        v, sample, dt, epi = cpu_reference(cfg, per_step, threads)
        if i >= args.warmup:
            vals.append((v, dt))
    value = float(np.mean([v for v, _ in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean([dt for _, dt in vals]) * 1e3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded mesh)",
        "config": {**cfg.describe(), "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)



_KERNEL_OF_PHASE = {"pair_full": "k_full", "pair_clipped": "k_clipped", "touching_singular": "k_singular"}


def _ncu_traffic(phase, config):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the
    newest committed `ncu --set full` summary of config 2 (profiles/); None
    for other configs or when no summary exists."""
    import glob
    import re
    if config != 2:
        return None, None
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                          f"r*_{_KERNEL_OF_PHASE[phase]}_ncu_summary.txt")))
    if not files:
        return None, None
    txt = open(files[-1]).read()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    total = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m = re.search(rf"^{re.escape(key)}\s+([0-9.]+) (\w+)", txt, re.M)
        if not m:
            return None, None
        total += float(m.group(1)) * scale.get(m.group(2), 1)
    return total, os.path.relpath(files[-1], os.path.dirname(os.path.abspath(__file__)))

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--emulate-shard", default=None, metavar="R/W",
                    help="single GPU: time only the rows rank R of W would own (a per-rank projection "
                         "for meshes whose CSR does not fit one GPU, e.g. config 4)")
    args = ap.parse_args()
    ws, rank, local = dist_env()

    from paper_2207_03921_b200 import configs
    cfg = configs.build(args.config)
    if args.impl == "reference":
        run_reference(args, cfg, ws, rank)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    from paper_2207_03921_b200 import _native, bfs_assemble
    from paper_2207_03921_b200.assembly import DevicePlan
    from paper_2207_03921_b200.problem import marshal

    inp = marshal(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad)
    J = inp.n_dofs
    from paper_2207_03921_b200 import shard
    srank, sws = rank, ws
    if args.emulate_shard and ws == 1:
        srank, sws = (int(x) for x in args.emulate_shard.split("/"))
    lo, hi = shard.my_rows(J, inp.nc, srank, sws, shard.vertex_work(cfg.mesh, cfg.ansatz))
    plan = DevicePlan(inp, device=local, on_device=True)  # mesh arrays resident in HBM
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")  # > 126 MB L2

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        plan.assemble(lo, hi, out_on_host=False, reuse_output=True)
    barrier()
    launches0 = _native.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    with ClockSampler(local) as clk:
        barrier()
        for i in range(args.steps):
            flush.fill_(float(i))  # evict L2 between steps (outside the timed pair)
            ev[i][0].record()
            _, _, _, st = plan.assemble(lo, hi, out_on_host=False, reuse_output=True)
            ev[i][1].record()
            stats.append(st)
        barrier()
    launches = _native.launch_count() - launches0 - 0  # our kernels + CUB passes (fill_ is torch's)
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    t_local = float(sum(ms_steps))
    epi_local = float(np.mean([s["epi"] for s in stats]))
    if dist is not None:
        t = torch.tensor([t_local, epi_local], dtype=torch.float64, device=f"cuda:{local}")
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        esum = t[1:].clone()
        dist.all_reduce(esum, op=dist.ReduceOp.SUM)
        t_total, epi_total = float(tmax.item()), float(esum.item())
    else:
        t_total, epi_total = t_local, epi_local
    ms_per_step = t_total / args.steps
    value = epi_total / (ms_per_step * 1e-3)

    # ---- roofline of the dominant integration kernel (live CUDA-event phase times)
    st0 = stats[-1]
    phases = {"pair_full": ("ms_full", "alg_flops_full"), "pair_clipped": ("ms_partial", "alg_flops_partial"),
              "touching_singular": ("ms_singular", "alg_flops_singular")}
    avg = {k: float(np.mean([s[v[0]] for s in stats])) for k, v in phases.items()}
    dom = max(avg, key=avg.get)
    peak_fp64 = _native.fp64_peak_tflops(local)
    dom_ms = avg[dom]
    dom_flops = st0[phases[dom][1]]
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12 if dom_ms > 0 else 0.0
    integ_ms = float(np.mean([s["ms_integrate_kernels"] for s in stats]))
    traffic, traffic_src = _ncu_traffic(dom, args.config)
    roofline = {
        "bound": "fp64", "kernel": dom, "achieved": achieved, "peak": peak_fp64, "unit": "TFLOP/s",
        "frac": achieved / peak_fp64 if peak_fp64 else None, "traffic": traffic, "traffic_source": traffic_src,
        "peak_source": "measured DFMA microbenchmark (nlg_fp64_peak) on this GPU, this run",
        "alg_flops_per_launch": dom_flops, "kernel_ms": dom_ms,
        "all_integration": {"alg_flops": st0["alg_flops"], "ms": integ_ms,
                            "tflops": st0["alg_flops"] / (integ_ms * 1e-3) / 1e12 if integ_ms else 0.0},
        "phase_ms": {k: float(np.mean([s[k] for s in stats])) for k in
                     ("ms_prep", "ms_candidates", "ms_full", "ms_partial", "ms_singular", "ms_merge", "ms_merge_stage_r", "ms_total")},
        "merge_hbm": {"coo_entries": st0["coo_entries"], "coo_reduced": st0["coo_reduced"], "nnz": st0["nnz"]},
        "batches": {"n": st0["n_batches"], "replans": st0["n_replans"], "row_retries": st0["n_row_retries"],
                    "merge_fallbacks": st0["n_merge_fallbacks"]},
    }
    # the merge (stage W) against HBM: algorithmic bytes = the stored record
    # values it reads once (8 B each) + the CSR it writes (12 B per entry);
    # analytic full pairs read only per-element factors (L2-resident)
    merge_ms = float(np.mean([s["ms_merge"] for s in stats]))
    merge_bytes = 8.0 * st0["coo_entries"] + 12.0 * st0["nnz"]
    hbm_peak = _peaks().get("hbm_gbs")
    roofline["merge"] = {
        "bound": "hbm", "alg_bytes": merge_bytes, "ms": merge_ms,
        "achieved_gbs": merge_bytes / (merge_ms * 1e-3) / 1e9 if merge_ms else None,
        "peak_gbs": hbm_peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if hbm_peak else None,
        "frac": (merge_bytes / (merge_ms * 1e-3) / 1e9) / hbm_peak if (merge_ms and hbm_peak) else None,
        "note": "shared-memory atomic / latency bound (stage W hash tables), not HBM bound",
    }

    # ---- end to end through the public API (host numpy in, host scipy CSR out)
    e2e = None
    if not args.no_e2e:
        h2d = sum(a.nbytes for a in (inp.vertices, inp.elements, inp.labels, inp.outer_mask, inp.dof_map))
        times, d2h = [], 0
        for i in range(max(1, min(args.steps, 3)) + 1):
            barrier()
            t0 = time.perf_counter()
            sysm = bfs_assemble(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad,
                                device=local, row_range=(lo, hi))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if i:
                times.append(dt)
            d2h = (hi - lo + 1) * 8 + sysm.matrix.nnz * 12  # int64 indptr, int32 indices, f64 data
        tl = float(np.mean(times))
        if dist is not None:
            t = torch.tensor([tl], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tl = float(t.item())
        e2e = {"value": epi_total / tl, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": tl * 1e3}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        v, sample, dt, _ = cpu_reference(cfg, args.ref_seconds, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
               "seconds": dt}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mesh, SURVEY.md App. A)",
            "config": {**cfg.describe(), "epi": epi_total,
                       "rows": "all" if (lo, hi) == (0, J) else f"[{lo}, {hi}) of {J}",
                       "parallelism": f"rowshard{ws}" if sws == ws else f"emulated rank {srank} of {sws} on 1 GPU",
                       "l2": "flushed between steps (512 MB write)", "inputs": "mesh arrays resident in HBM",
                       "output": "CSR resident in HBM"},
            "assembly_ms": ms_per_step,
            "step_ms": [round(x, 3) for x in ms_steps],
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    plan.close()


if __name__ == "__main__":
    main()
