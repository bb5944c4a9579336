"""Benchmark: full nonlocal stiffness assembly (fp64) on B200 vs the CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]
    python bench.py --config 4 --emulate-shards 8     # config 4 on one GPU, rank by rank

A step is one complete assembly of BASELINE config C from mesh arrays
resident in HBM to the CSR resident in HBM: element bounds, grid hash,
candidate search, pair integration, touching-pair tensor rules and the row
merge into CSR.  The default is config 5 (the N=512 jittered L-shape with
the nonsymmetric kernel, 4.87e9 EPI): the largest configuration whose CSR
fits one GPU (config 4's ~266 GB CSR does not; ``--emulate-shards 8`` times
its eight row shards one after the other on one GPU instead).  ``value`` =
evaluated element-pair integrals (EPI) / second over the whole
job.  ``e2e`` repeats the step through the public drop-in API
``bfs_assemble`` with host numpy inputs and a host scipy CSR out (H2D and
D2H inside the timed region).

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


def cpu_path_label(cfg, kernel=None):
    """What the CPU oracle restates for this config's kernel (the reference's
    own path for it)."""
    kid = int((kernel or cfg.kernel).builtin_id)
    if kid == 3:
        return ("C restatement (oracle/, bit-identical) of the reference's interpreted engine "
                "(_pyengine, the only reference path for the nonsymmetric kernel) + _merge_triplets")
    return "C restatement (oracle/, bit-identical) of the reference's numba engine (_engine._chunk) + _merge_triplets"


def cpu_reference(cfg, budget_s, threads, kernel=None):
    """The reference algorithm (oracle port, bit-identical) on a bounded band
    of outer elements: returns EPI/s, the sample description and seconds.
    ``kernel`` replaces the config's kernel (the symmetric-constant proxy of
    config 5)."""
    from oracle import oracle
    from paper_2207_03921_b200.problem import marshal
    inp = marshal(cfg.mesh, cfg.adjacency, kernel or cfg.kernel, cfg.ansatz, cfg.quad)
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


def cpu_baselines(cfg, budget_s, threads):
    """cpu_baseline of the line: the reference's path for the config's kernel
    on a bounded sample; config 5 adds the compiled-engine proxy (symmetric
    constant kernel on the same mesh), both labelled."""
    v, sample, dt, _ = cpu_reference(cfg, budget_s, threads)
    out = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample, "seconds": dt,
           "path": cpu_path_label(cfg), "cpu_model": cpu_model()}
    if int(cfg.kernel.builtin_id) == 3:
        from paper_2207_03921_b200.kernels import constant_kernel
        proxy = constant_kernel(cfg.kernel.delta, cfg.kernel.ball)
        pv, psample, pdt, _ = cpu_reference(cfg, budget_s / 2, threads, kernel=proxy)
        out["proxy"] = {"value": pv, "unit": UNIT, "cores": threads, "sample": psample, "seconds": pdt,
                        "path": cpu_path_label(cfg, proxy) + "; symmetric constant kernel (id 2) on the same mesh",
                        "note": "the reference's compiled engine cannot evaluate the nonsymmetric kernel"}
    return out


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
                         "sample": sample, "path": cpu_path_label(cfg), "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)



def merge_alg_bytes(cfg, inp, st):
    """Algorithmic HBM bytes of the merge (stage W, k_row_asm) per assembly:
    every stored record-side block read once (own block NKK + neighbour block
    9 nc^2 values of 8 B: 6 + 9 = 15 for nc = 1), the touching-pair COO
    (16 B per slot), the record lists (8 B per record), the per-element
    tables once (element, dofs, analytic factors: 64 B per element) and the
    CSR written (int32 column + f64 value per entry, int64 row pointers)."""
    nc = inp.nc
    nkk, nkl = 3 * nc * (3 * nc + 1) // 2, 9 * nc * nc
    analytic = inp.kernel_id in (2, 3) and inp.path_touch == 0 and nc == 1
    stored = st["n_partial"] + (0 if analytic else st["n_full"])
    blocks = 2 * stored * (nkk + nkl) * 8
    sing = st["n_singular"] * 36 * nc * nc * 16
    lists = (st["n_full"] + st["n_partial"]) * 8
    tables = inp.elements.shape[0] * 64
    csr = st["nnz"] * 12 + (inp.n_dofs + 1) * 8
    return {"stored_blocks": blocks, "singular_coo": sing, "record_lists": lists, "element_tables": tables,
            "csr_out": csr, "total": float(blocks + sing + lists + tables + csr)}


def _ncu_traffic(kernel, config):
    """(DRAM bytes read + written, source file, extras) of ONE launch of
    ``kernel`` from the newest committed `ncu --set full` summary of this
    config under profiles/ (r*_cfg<C>_<kernel>_ncu_summary.txt); a step runs
    one launch per row batch.  (None, None, {}) when no capture exists."""
    import glob
    import re
    here = os.path.dirname(os.path.abspath(__file__))
    files = sorted(glob.glob(os.path.join(here, "profiles", f"r*_cfg{config}_{kernel}_ncu_summary.txt")) +
                   glob.glob(os.path.join(here, "profiles", f"r*_{kernel}_cfg{config}_ncu_summary.txt")),
                   key=lambda f: os.path.basename(f).split("_")[0])
    if not files:
        return None, None, {}
    txt = open(files[-1]).read()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    total = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m = re.search(rf"^{re.escape(key)}\s+([0-9.]+) (\w+)", txt, re.M)
        if not m:
            return None, None, {}
        total += float(m.group(1)) * scale.get(m.group(2), 1)
    extra = {}
    for key, name in (("gpu__time_duration.sum", "launch_ms"),
                      ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_active_pct"),
                      ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue_active_pct"),
                      ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
                      ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_instruction")):
        m = re.search(rf"^{re.escape(key)}\s+([0-9.]+)", txt, re.M)
        if m:
            extra[name] = float(m.group(1))
    return total, os.path.relpath(files[-1], here), extra


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_emulated_shards(args, cfg):
    """Every rank's row shard of the config, one after the other on this GPU
    (owner computes: each shard evaluates the outer elements reaching its
    rows, no collective).  T1 = sum of the shard times is the full 1-GPU
    assembly (streamed by shard; config 4's whole CSR does not fit one GPU),
    max_r T_r the W-GPU time.  Each shard's CSR gets a device checksum."""
    import torch
    from paper_2207_03921_b200 import _native, shard
    from paper_2207_03921_b200.assembly import DevicePlan
    from paper_2207_03921_b200.problem import marshal
    torch.cuda.set_device(0)
    inp = marshal(cfg.mesh, cfg.adjacency, cfg.kernel, cfg.ansatz, cfg.quad)
    W = args.emulate_shards
    plan = DevicePlan(inp, device=0, on_device=True)
    weights = shard.row_weights(plan, cfg.mesh, cfg.ansatz)
    cuts = shard.row_partition(inp.n_dofs, inp.nc, W, weights)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
    launches0 = _native.launch_count()
    shards = []
    with ClockSampler(0) as clk:
        for r in range(W):
            lo, hi = cuts[r], cuts[r + 1]
            for _ in range(args.warmup if r == 0 else 1):
                plan.assemble(lo, hi, out_on_host=False, reuse_output=True)
            times, epi = [], 0
            for i in range(args.steps):
                flush.fill_(float(i))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                ip, ix, dv, st = plan.assemble(lo, hi, out_on_host=False, reuse_output=True)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
                epi = st["epi"]
            nnz = int(st["nnz"])
            chk = {"nnz": nnz, "sum_data": float(dv[:nnz].sum().item()),
                   "sum_abs_data": float(dv[:nnz].abs().sum().item()),
                   "sum_indices": int(ix[:nnz].to(torch.int64).sum().item())}
            shards.append({"rank": r, "rows": [lo, hi], "ms": float(np.mean(times)), "epi": int(epi),
                           "batches": st["n_batches"], "checksum": chk,
                           "phase_ms": {k: st[k] for k in ("ms_candidates", "ms_partial", "ms_merge")}})
            print(json.dumps({"shard": shards[-1]}), file=sys.stderr, flush=True)
    t1 = sum(x["ms"] for x in shards)
    tmax = max(x["ms"] for x in shards)
    epi = sum(x["epi"] for x in shards)
    line = {
        "metric": METRIC, "value": epi / (t1 * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t1, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded mesh, SURVEY.md App. A)",
        "config": {**cfg.describe(), "epi": epi, "rows": "all, as %d row shards run one after the other" % W,
                   "parallelism": f"{W} emulated row shards on 1 GPU", "l2": "flushed between steps (512 MB write)",
                   "inputs": "mesh arrays resident in HBM", "output": "each shard's CSR resident in HBM in turn"},
        "assembly_ms": t1,
        "projected": {"n_gpus": W, "max_rank_ms": tmax, "efficiency": t1 / (W * tmax),
                      "note": "T1 / (W max_r T_r): per-rank work measured on one GPU; no collective on the data path"},
        "shards": shards, "gpu_launches": int(_native.launch_count() - launches0), "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    plan.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--emulate-shards", type=int, default=0, metavar="W",
                    help="single GPU: time the row shards of all W ranks one after the other (config 4: the "
                         "1-GPU full-assembly time T1 = their sum, and the projected W-GPU efficiency "
                         "T1 / (W max_r T_r))")
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
    if args.emulate_shards:
        run_emulated_shards(args, cfg)
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
    plan = DevicePlan(inp, device=local, on_device=True)  # mesh arrays resident in HBM
    # rows balanced by EPI prefix sums, from the device's count pass
    lo, hi = (0, J) if sws == 1 else shard.my_rows(J, inp.nc, srank, sws, shard.row_weights(plan))
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")  # > 126 MB L2

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # Row batches: the library plans a batch within 60 % of the device by
    # default.  This process holds nothing else on the GPU, so the timed steps
    # allow 75 % -- config 5 then runs as ONE batch and no pair is integrated
    # twice at a batch cut (768 vs 825 ms).  The warm-up proves it fits; if it
    # does not, the library default is used.  (e2e below: library defaults.)
    # (whole problems only: a config-4 shard at 75 % ran out of memory)
    budget = int(0.75 * torch.cuda.mem_get_info(local)[1]) if sws == 1 else 0
    try:
        for _ in range(args.warmup):
            plan.assemble(lo, hi, out_on_host=False, reuse_output=True, mem_budget=budget)
    except Exception as exc:  # noqa: BLE001
        print(f"# mem_budget 75 % did not fit ({exc}); library default", file=sys.stderr)
        budget = 0
        torch.cuda.empty_cache()
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
            _, _, _, st = plan.assemble(lo, hi, out_on_host=False, reuse_output=True, mem_budget=budget)
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

    # ---- roofline: every timed phase against its bound; the top-level line
    # is the dominant (longest) phase's kernel
    st0 = stats[-1]
    phase_avg = {k: float(np.mean([s[k] for s in stats])) for k in
                 ("ms_prep", "ms_candidates", "ms_full", "ms_partial", "ms_singular", "ms_merge", "ms_merge_stage_r",
                  "ms_total")}
    peak_fp64 = _native.fp64_peak_tflops(local)
    hbm_peak = _peaks().get("hbm_gbs")
    phases = {}
    for name, ms_key, fl_key in (("k_full", "ms_full", "alg_flops_full"), ("k_clipped", "ms_partial", "alg_flops_partial"),
                                 ("k_singular", "ms_singular", "alg_flops_singular")):
        ms = phase_avg[ms_key]
        ach = st0[fl_key] / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
        phases[name] = {"bound": "fp64", "ms": ms, "alg_flops": st0[fl_key], "achieved": ach, "peak": peak_fp64,
                        "unit": "TFLOP/s", "frac": ach / peak_fp64 if peak_fp64 else None}
    mb = merge_alg_bytes(cfg, inp, st0)
    ms = phase_avg["ms_merge"]
    phases["k_row_asm"] = {"bound": "hbm", "ms": ms, "alg_bytes": mb["total"], "bytes_model": mb,
                           "achieved": mb["total"] / (ms * 1e-3) / 1e9 if ms else None, "peak": hbm_peak,
                           "unit": "GB/s", "frac": (mb["total"] / (ms * 1e-3) / 1e9) / hbm_peak if (ms and hbm_peak) else None}
    phases["k_candidates"] = {"bound": "l2/latency", "ms": phase_avg["ms_candidates"],
                              "note": "grid scan + exact reject/full/truncation-class tests per candidate (two passes)"}
    dom = max(phases, key=lambda k: phases[k]["ms"])
    top = phases[dom] if phases[dom].get("frac") is not None else phases["k_clipped"]
    dom_name = dom if phases[dom].get("frac") is not None else "k_clipped"
    # (the clipped pairs of the constant / affine kernels run in k_clipped_cfr)
    closed_form = inp.kernel_id in (2, 3) and inp.path_touch == 0 and inp.ball_id != 2
    kern_name = "k_clipped_cfr" if dom_name == "k_clipped" and closed_form else dom_name
    traffic, traffic_src, ncu_extra = _ncu_traffic(kern_name, args.config)
    roofline = {
        "bound": top["bound"], "kernel": kern_name, "achieved": top["achieved"], "peak": top["peak"], "unit": top["unit"],
        "frac": top["frac"], "traffic": traffic, "traffic_source": traffic_src,
        "traffic_note": "DRAM bytes of ONE launch (ncu --set full); a step runs one launch per row batch",
        "ncu": ncu_extra,
        "peak_source": ("measured DFMA microbenchmark (nlg_fp64_peak) on this GPU, this run" if top["bound"] == "fp64"
                        else "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"),
        "kernel_ms": top["ms"], "share_of_step": top["ms"] / ms_per_step if ms_per_step else None,
        "dominant_phase": dom,
        "phases": phases,
        "all_integration": {"alg_flops": st0["alg_flops"], "ms": float(np.mean([s["ms_integrate_kernels"] for s in stats])),
                            "note": "reference-algorithmic flops (SURVEY 8d) of all integration kernels"},
        "phase_ms": phase_avg,
        "batches": {"n": st0["n_batches"], "replans": st0["n_replans"], "row_retries": st0["n_row_retries"],
                    "merge_fallbacks": st0["n_merge_fallbacks"]},
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
            del sysm  # (its page-locked block goes back to the pool for the next step)
        tl = float(np.mean(times))
        if dist is not None:
            t = torch.tensor([tl], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tl = float(t.item())
        e2e = {"value": epi_total / tl, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": tl * 1e3}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baselines(cfg, args.ref_seconds, len(os.sched_getaffinity(0)))

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
                       "output": "CSR resident in HBM",
                       "mem_budget": "75 % of HBM per row batch" if budget else "library default (60 %)"},
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
