#!/usr/bin/env python
"""Benchmark: Helmholtz solves/s to 1e-6 relative residual (BASELINE.json metric)
through the B200 FGMRES + shifted-Laplacian multigrid (+ U-Net) hot path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c0] [--replicas R]

Workload: config c0 -- 128^2 heterogeneous
Helmholtz, unit point source, M_V (3-level shifted-Laplacian V-cycle, GMRES(10)
coarsest), FGMRES(10) to 1e-6.  It is the only BASELINE config whose solve
reaches 1e-6 with the seeded random-init weights the configs prescribe (c1-c4
put a random-init U-Net in the preconditioner and stagnate; the oracle shows
it).  One step = R independent c0 solves on one GPU, R = 6 per SM
(888) by default -- two columns per SM in each of the 3 column groups, the
device-filling analog of the reference arm, which runs one c0 solve per host
core (throughput saturates there; round 2, device / end to end: 296 -> 11.5k /
10.6k, 444 -> 12.5k / 11.9k, 666 -> 12.8k / 12.3k, 888 -> 13.0k / 12.5k,
1776 -> 13.2k / 12.8k solves/s).  Inputs resident in HBM; the per-step working
set (~3 GB) exceeds L2, and L2 is additionally flushed (512 MiB write) between
timed steps.  Multi-GPU: each rank runs its own R replicas (weak scaling, no
collective).  The U-Net configs are measured on a fixed iteration budget under
"also".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the C oracle's OpenMP threads (CPU reference legs) must not spin on the host
# cores the device path's host work (e.g. training-pair draws) needs afterwards
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

METRIC = "Helmholtz solves/s to 1e-6 rel residual"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


def tf32_peak():
    """Dense tcgen05 kind::tf32 peak measured on this B200 pool by
    tools/micro/tf32_peak.cu (profiles/tf32_peak.json: M=128, N=256, K=8 SS
    MMAs on every SM, event-timed); fallback 0.5 x the measured bf16 peak."""
    try:
        with open(os.path.join(ROOT, "profiles", "tf32_peak.json")) as f:
            runs = json.load(f)["runs"]
        return max(r["tflops"] for r in runs), "measured (profiles/tf32_peak.json, tools/micro/tf32_peak.cu)"
    except Exception:
        pk, src = peaks()
        return 0.5 * pk.get("bf16_tflops", 1590.0), f"provisional 0.5 x {src} bf16"


E2E_STAGGER_S = 0.003  # start offset between column groups in the pipelined e2e loop (> one group's copies)


# ------------------------------------------------------------------ dist
def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            time.sleep(0.2)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- workloads
def config_for(name):
    from paper_2203_11025_b200 import configs
    return dict(configs.CONFIGS[name])


def columns(cfg, ws, rank, replicas):
    """RHS of this rank: the config's own RHS block sharded by rank (
    uneven world sizes get contiguous np.array_split shards, a rank beyond B gets
    none), or R replicas of a single-RHS config."""
    B = cfg["B"]
    if B > 1:
        return [int(c) for c in np.array_split(np.arange(B), ws)[rank]]
    return [0] * replicas


def sum_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def make_solver(O, kind, cfg, arr):
    mk = O.RefHierarchy if kind == "reference" else O.Hierarchy
    H = mk(arr["kappa2"], arr["gamma"], arr["omega"], arr["lo"], arr["hi"], levels=cfg["levels"],
           coarse=cfg["coarse"], coarse_iters=cfg["coarse_iters"])
    P = (O.RefPrecond if kind == "reference" else O.Precond)("v", H)
    solve = O.ref_fgmres if kind == "reference" else O.fgmres
    return H, P, solve


def ref_config(name):
    """Config table for the CPU legs, loaded without importing the product."""
    from oracle import problems as OP
    return dict(OP.configs().CONFIGS[name])


def cpu_baseline_sample(cfg_name, cfg):
    """The reference CPU path (oracle/_ref: the reference headers compiled in place)
    on a bounded sample: one full solve, one thread.  Falls back to the C
    restatement ('port') if the reference build is absent.  Inputs come from the
    oracle's generators (oracle/problems.py), bit-identical to the product's."""
    from oracle import oracle as O
    from oracle import problems as OP
    arr = OP.problem_arrays(cfg)
    B = OP.rhs_block(arr)[:1]
    kind = "reference" if O.have_ref() else "port"
    H, P, solve = make_solver(O, kind, cfg, arr)
    # repeated full solves until ~10 s of CPU work (bounded sample)
    n, t0 = 0, time.perf_counter()
    while True:
        X, rep = solve(P, B, restart=cfg["restart"], max_iters=cfg["max_iters"], nthreads=1)
        n += 1
        dt = time.perf_counter() - t0
        if dt >= 10.0 or n >= 500:
            break
    return {"value": n / dt, "unit": "solves/s", "cores": 1, "kind": kind, "cpu": cpu_model(),
            "sample": f"{n} full {cfg_name} solves ({int(rep['iterations'][0])} FGMRES iterations each, "
                      f"converged={bool(rep['converged'][0])}) on 1 host thread, {dt:.2f} s"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cpus)"
    except OSError:
        pass
    return None


# full-solve iteration counts used to extrapolate fixed-budget CPU times (BASELINE.md
# 4.4): the reference's converged M_V counts on the BASELINE medium;
# c4 is the survey's extrapolation (~1e4).  Labelled "extrapolated" in the output.
MV_ITERS_FULL = {"c1": 346, "c2": 795, "c3": 1885, "c4": 10000}


def cpu_reference_budget(name, iters):
    """The reference CPU path on a fixed FGMRES budget of one column of config
    `name` (1 host thread): seconds per iteration, plus a full-solve time
    extrapolated with MV_ITERS_FULL (labelled as such)."""
    from oracle import oracle as O
    from oracle import problems as OP
    cfg = ref_config(name)
    arr = OP.problem_arrays(cfg)
    kind = "reference" if O.have_ref() else "port"
    t0 = time.perf_counter()
    H, P = ref_preconditioner(O, kind, cfg, arr)
    setup = time.perf_counter() - t0
    B = OP.rhs_block(arr)[:1]
    solve = O.ref_fgmres if kind == "reference" else O.fgmres
    t0 = time.perf_counter()
    X, rep = solve(P, B, restart=cfg["restart"], max_iters=iters, nthreads=1)
    dt = time.perf_counter() - t0
    its = max(1, int(rep["iterations"][0]))
    out = {"kind": kind, "cores": 1, "cpu": cpu_model(), "iterations": its, "s": dt,
           "ms_per_iteration": 1e3 * dt / its, "setup_s": setup,
           "sample": f"{its} FGMRES iterations of 1 {name} column on 1 host thread"}
    if name in MV_ITERS_FULL:
        out["extrapolated_solve_s"] = dt / its * MV_ITERS_FULL[name]
        out["extrapolation"] = (f"ms_per_iteration x {MV_ITERS_FULL[name]} iterations (the reference M_V count "
                                "at this grid, SURVEY App. B) -- extrapolated, not measured")
    del H, P
    return out


def ref_preconditioner(O, kind, cfg, arr):
    """Hierarchy + preconditioner of config cfg on the CPU side (reference build or
    the C restatement), including the config's nets with the same He seeds."""
    pre = "Ref" if kind == "reference" else ""
    Net = O.RefNet if kind == "reference" else O.UNet
    net = enc = None
    if cfg["net"] is not None:
        L, base, seed, ctx_ch = cfg["net"]
        net = Net(0, L, base, 3, ctx_ch, seed=seed)
    if cfg["enc"] is not None:
        L, base, seed = cfg["enc"]
        enc = Net(1, L, base, 1, 0, seed=seed)
    Hc = getattr(O, pre + "Hierarchy")
    coarse_net = net if cfg["coarse"] == "net" else None
    H = Hc(arr["kappa2"], arr["gamma"], arr["omega"], arr["lo"], arr["hi"], levels=cfg["levels"],
           coarse=cfg["coarse"], coarse_iters=max(1, cfg["coarse_iters"]), coarse_net=coarse_net)
    P = getattr(O, pre + "Precond")(cfg["precond"], H, net=net if cfg["precond"] != "v" else None, enc=enc)
    P._keep = (net, enc, H)
    return H, P


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref) on all
    host threads, one c0 solve per thread per step (replicas, as our arm).  Inputs
    from the oracle's generators: this process never loads libhelmgpu.so."""
    if rank != 0:
        return
    from oracle import oracle as O
    from oracle import problems as OP
    cfg = ref_config(args.config)
    arr = OP.problem_arrays(cfg)
    Bfull = OP.rhs_block(arr)
    threads = os.cpu_count() or 1
    kind = "reference" if O.have_ref() else "port"
    H, P, solve = make_solver(O, kind, cfg, arr)
    cols = np.stack([Bfull[i % Bfull.shape[0]] for i in range(threads)])
    times, conv, iters = [], [], []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        X, rep = solve(P, cols, restart=cfg["restart"], max_iters=cfg["max_iters"], nthreads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            conv.append(bool(np.all(rep["converged"])))
            iters.append(int(np.max(rep["iterations"])))
    total = sum(times)
    value = threads * args.steps / total
    line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (fp64), fp32 network",
            "data": "synthetic (seeded media / point sources, SURVEY 8(d))", "impl": "reference",
            "config": {"workload": args.config, "grid": cfg["n"], "rhs_per_step": threads,
                       "iterations": iters[-1] if iters else None, "converged": all(conv),
                       "note": "one independent solve per host thread per step; inputs from oracle/problems.py"},
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": kind, "cpu": cpu_model(),
                             "sample": f"{threads} concurrent {args.config} solves per step x {args.steps} steps"},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def ncu_traffic(kernel_class):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    dominant kernel class, from the committed ncu --set full capture of the same
    bench command (profiles/ncu_traffic.json, written by tools/ncu_traffic.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        e = t["classes"][kernel_class]
        return {"bytes_per_launch": e["dram_bytes_per_launch"], "source": t["source"]}
    except Exception:
        return None


def run_ours(args, ws, rank, local):
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    from paper_2203_11025_b200 import problems
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cfg = config_for(args.config)
    R = args.replicas or 6 * sms
    cols = columns(cfg, ws, rank, R)
    # G column groups = G independent solver contexts on their own streams, driven
    # from G host threads: one group's latency-bound coarsest solves overlap the
    # other's bandwidth-bound legs / Krylov kernels
    G = max(1, min(args.groups, len(cols) // 16 or 1))
    bounds = [len(cols) * g // G for g in range(G + 1)]
    groups = []
    for g in range(G):
        cg, arr = problems.gpu_setup(cfg, device=local)
        for kv in args.opt:  # library options (experiments), e.g. --opt pdl=0
            k, v = kv.split("=")
            cg.set_option(k, int(v))
        groups.append(cg)
    ctx = groups[0]
    Bh = np.ascontiguousarray(problems.rhs_block(arr)[cols])
    nb = Bh.shape[0]
    kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=cfg["max_iters"], rel_tol=1e-6)
    kind = cfg["precond"]
    dB = torch.from_numpy(Bh).to(dev)
    dX = torch.zeros_like(dB)
    streams = [torch.cuda.ExternalStream(cg.stream, device=dev) for cg in groups]
    stream = streams[0]
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)

    def run_groups(fn):
        """fn(g) for every group from its own host thread; returns the results"""
        out = [None] * G
        def body(g):
            out[g] = fn(g)
        th = [threading.Thread(target=body, args=(g,)) for g in range(1, G)]
        for t in th:
            t.start()
        body(0)
        for t in th:
            t.join()
        return out

    def solve_group(g, report=False):
        lo, hi = bounds[g], bounds[g + 1]
        return groups[g].fgmres_device(kind, dB[lo:hi].data_ptr(), dX[lo:hi].data_ptr(), hi - lo, kc,
                                       want_report=report)

    def timed(fn):
        """device time of fn() over all group streams: start event on stream 0 (the
        others wait on it), end = the latest stream"""
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in streams[1:]:
            st.wait_event(e0)
        fn()
        ends = []
        for st in streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            ends.append(e)
        return e0, ends

    for _ in range(args.warmup):
        dX.zero_()
        run_groups(lambda g: solve_group(g))
    dX.zero_()
    reps = run_groups(lambda g: solve_group(g, report=True))
    torch.cuda.synchronize()
    rep = hg.SolveReport(sum((r.residual_history for r in reps), []), sum((r.iterations for r in reps), []),
                         sum((r.converged for r in reps), []), sum((r.breakdown for r in reps), []))

    # ---- timed region: K steps, CUDA events on the library streams, L2 flushed between steps
    barrier(ws)
    torch.cuda.synchronize()
    n0 = sum(cg.launch_count() for cg in groups)
    marks = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.add_(1.0)
            dX.zero_()
            torch.cuda.synchronize()
            marks.append(timed(lambda: run_groups(lambda g: solve_group(g))))
        torch.cuda.synchronize()
    launches = (sum(cg.launch_count() for cg in groups) - n0) // max(1, args.steps)
    t_ms = sum(max(e0.elapsed_time(e) for e in ends) for e0, ends in marks)
    barrier(ws)
    t_ms = max_over_ranks(t_ms, ws)
    solves = sum_over_ranks(nb, ws) * args.steps  # distinct RHS over all ranks (uneven shards allowed)
    value = solves / (t_ms / 1e3)

    # ---- e2e: the public C ABI (hb_fgmres) on pinned host buffers; H2D of B and
    # D2H of X inside the timed region every step
    Bpin = torch.from_numpy(Bh).pin_memory()
    Xpin = torch.zeros_like(Bpin).pin_memory()
    Bn, Xn = Bpin.numpy(), Xpin.numpy()
    # warm-up of this path (its staging buffers are allocated on first use, which
    # re-captures the restart-cycle graphs)
    run_groups(lambda g: groups[g].fgmres(kind, Bn[bounds[g]:bounds[g + 1]], kc, out=Xn[bounds[g]:bounds[g + 1]]))
    torch.cuda.synchronize()
    emarks = []
    for k in range(args.steps):
        flush.add_(1.0)
        torch.cuda.synchronize()
        emarks.append(timed(lambda: run_groups(
            lambda g: groups[g].fgmres(kind, Bn[bounds[g]:bounds[g + 1]], kc, out=Xn[bounds[g]:bounds[g + 1]]))))
    torch.cuda.synchronize()
    e_ms = max_over_ranks(sum(max(e0.elapsed_time(e) for e in ends) for e0, ends in emarks), ws)
    e2e = {"value": solves / (e_ms / 1e3), "unit": "solves/s", "h2d_bytes_per_step": int(Bh.nbytes),
           "d2h_bytes_per_step": int(Bh.nbytes), "path": f"hb_fgmres (pinned host c128 buffers), {G} column groups",
           "mode": "every step: all groups start together, device idle during the copies"}
    # The same K steps as a host would run them in production: every column group
    # loops its K hb_fgmres calls on its own thread and stream with no step-wide
    # join, group g starting g x 3 ms late, so one group's H2D / D2H runs under the
    # other groups' kernels.  Same calls, same bytes per step, one timed region
    # around all K steps (the Krylov bases of the groups, 3 x 213 MB, exceed L2).
    if G > 1 and not getattr(args, "no_pipeline", False):
        def loop_group(g):
            time.sleep(g * E2E_STAGGER_S)
            lo, hi = bounds[g], bounds[g + 1]
            for _ in range(args.steps):
                groups[g].fgmres(kind, Bn[lo:hi], kc, out=Xn[lo:hi])
        flush.add_(1.0)
        torch.cuda.synchronize()
        barrier(ws)
        e0, ends = timed(lambda: run_groups(loop_group))
        torch.cuda.synchronize()
        p_ms = max_over_ranks(max(e0.elapsed_time(e) for e in ends), ws)
        e2e["per_step_sync"] = {"value": e2e["value"], "ms_per_step": e_ms / args.steps}
        e2e["value"] = solves / (p_ms / 1e3)
        e2e["ms_per_step"] = p_ms / args.steps
        e2e["mode"] = (f"pipelined: each of the {G} column groups loops its {args.steps} hb_fgmres calls on its own "
                       f"host thread and stream, starts staggered by {E2E_STAGGER_S * 1e3:.0f} ms; per_step_sync = "
                       "the same calls joined after every step")
    d_g0 = (dB[bounds[0]:bounds[1]], dX[bounds[0]:bounds[1]], bounds[1] - bounds[0])

    # ---- single-solve latency (R = 1)
    lat = None
    if cfg["B"] == 1:
        d1B, d1X = dB[:1].contiguous(), torch.zeros_like(dB[:1])
        for _ in range(2):
            d1X.zero_()
            ctx.fgmres_device(kind, d1B.data_ptr(), d1X.data_ptr(), 1, kc)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d1X.zero_()
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.fgmres_device(kind, d1B.data_ptr(), d1X.data_ptr(), 1, kc, want_report=False)
        e1.record(stream)
        torch.cuda.synchronize()
        lat = e0.elapsed_time(e1)

    # ---- roofline pass: same workload, per-kernel-class CUDA events on the library
    # stream (eager launches; the timed region above replays CUDA graphs)
    # one column group, its two half-batch V-cycle streams serialised, so that
    # per-launch event times are not inflated by concurrently running kernels
    ctx.set_option("split_vcycle", 0)
    ctx.prof_reset()
    ctx.prof_enable(True)
    for _ in range(args.steps):
        d_g0[1].zero_()
        ctx.fgmres_device(kind, d_g0[0].data_ptr(), d_g0[1].data_ptr(), d_g0[2], kc, want_report=False)
    torch.cuda.synchronize()
    ctx.prof_enable(False)
    ctx.set_option("split_vcycle", 1)
    prof = ctx.prof()
    total_ms = sum(p["ms"] for p in prof.values()) or 1.0
    pk, src = peaks()
    kernels = {}
    for k, v in prof.items():
        if not v["launches"]:
            continue
        row = {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
               "share": v["ms"] / total_ms, "avg_launch_us": 1e3 * v["ms"] / v["launches"]}
        if v["flops"] > 0:
            row["tflops"] = v["flops"] / (v["ms"] / 1e3) / 1e12
        if v["bytes"] > 0:
            row["gbs"] = v["bytes"] / (v["ms"] / 1e3) / 1e9
            row["hbm_frac"] = row["gbs"] / pk.get("hbm_gbs", 6650.0)
        kernels[k] = row
    # BASELINE's second metric: precond-apply % of roofline -- the V-cycle classes
    # (legs + coarsest solve) per apply, algorithmic bytes vs HBM peak
    pcls = [k for k in ("vcycle_down", "vcycle_up", "coarse_solve", "smooth", "transfer") if prof.get(k, {}).get("launches")]
    n_apply = max(1, prof.get("coarse_solve", {}).get("launches", 0))
    pc_ms = sum(prof[k]["ms"] for k in pcls)
    pc_bytes = sum(prof[k]["bytes"] for k in pcls)
    precond_apply = {"classes": pcls, "applies": n_apply, "us_per_apply": 1e3 * pc_ms / n_apply,
                     "bytes_per_apply": pc_bytes / n_apply,
                     "gbs": pc_bytes / (pc_ms / 1e3) / 1e9 if pc_ms > 0 else 0.0}
    precond_apply["hbm_frac"] = precond_apply["gbs"] / pk.get("hbm_gbs", 6650.0)
    name, p = max(prof.items(), key=lambda kv: kv[1]["ms"])
    if p["flops"] > 0:
        achieved = p["flops"] / (p["ms"] / 1e3) / 1e12
        peak, tsrc = tf32_peak()
        rl = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
              "traffic": None, "kernel": name, "note": f"peak = tcgen05 kind::tf32 dense, {tsrc}; useful flops"}
    else:
        achieved = p["bytes"] / (p["ms"] / 1e3) / 1e9 if p["ms"] > 0 else 0.0
        peak = pk.get("hbm_gbs", 6650.0)
        rl = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
              "traffic": None, "kernel": name, "note": f"peak = {src} HBM copy bandwidth; algorithmic bytes per "
                                                       "launch as DESIGN.md 'Roofline accounting'"}
    if name == "coarse_solve":
        # the coarsest-level GMRES keeps its basis in registers / shared memory (1024 nodes per
        # column at c0): its algorithmic HBM bytes are f in and x out only, so the HBM roofline
        # does not bound it (it is latency-bound on chip: two CTA barriers and one reduce-scatter
        # per Arnoldi step).  The largest class the HBM roofline does bound is listed beside it.
        nm2, p2 = max(((k, v) for k, v in prof.items() if k != "coarse_solve" and v["bytes"] > 0 and v["ms"] > 0),
                      key=lambda kv: kv[1]["ms"], default=(None, None))
        rl["on_chip"] = True
        if nm2:
            a2 = p2["bytes"] / (p2["ms"] / 1e3) / 1e9
            rl["largest_hbm_bound_kernel"] = {"kernel": nm2, "achieved": a2, "frac": a2 / rl["peak"],
                                              "share_of_step": p2["ms"] / total_ms,
                                              "avg_launch_us": 1e3 * p2["ms"] / max(1, p2["launches"])}
            tr2 = ncu_traffic(nm2)
            if tr2 is not None:
                rl["largest_hbm_bound_kernel"]["traffic"] = tr2["bytes_per_launch"]
    rl["share_of_step"] = p["ms"] / total_ms
    rl["avg_launch_us"] = 1e3 * p["ms"] / max(1, p["launches"])
    tr = ncu_traffic(name)
    if tr is not None:
        rl["traffic"] = tr["bytes_per_launch"]
        rl["traffic_source"] = tr["source"]

    line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "complex64 fields (fp64 reductions/Hessenberg/solution), fp32 net",
            "data": "synthetic (seeded media / point sources, SURVEY 8(d))",
            "config": {"workload": args.config, "grid": cfg["n"], "rhs_per_gpu_per_step": nb,
                       "rhs_kind": "replicas of the single c0 RHS" if cfg["B"] == 1 else "config RHS block (sharded)",
                       "levels": cfg["levels"], "coarse": f"{cfg['coarse']}({cfg['coarse_iters']})",
                       "restart": cfg["restart"], "precond": kind, "iterations": int(max(rep.iterations)),
                       "all_converged": bool(all(rep.converged)),
                       "l2": "working set > L2; L2 flushed (512 MiB write) between steps",
                       "single_solve_latency_ms": lat, "column_groups_per_gpu": G,
                       "parallelism": f"independent solves x{ws} GPUs"},
            "roofline": rl, "kernels": kernels, "precond_apply": precond_apply, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample(args.config, cfg)
    for cg in groups:
        cg.close()
    also = [s for s in args.also.split(",") if s]
    slab, wedged = None, False
    if "c4slab" in also:  # every rank takes part (one slab per rank)
        # over NCCL (ws > 1) the slab exchange runs under a deadline: a wedged
        # collective must not take the headline line down with it
        slab, wedged = run_with_deadline(lambda: slab_budget(local, args, ws, rank), local,
                                         SLAB_DEADLINE_S if ws > 1 else None)
    if wedged:
        # the device may still be spinning in a collective: deliver the measured
        # line and leave without touching CUDA or the process group again
        if rank == 0:
            line["also"] = {nm: (slab if nm == "c4slab" else {"skipped": "after the c4slab deadline"}) for nm in also}
            print(json.dumps(line), flush=True)
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    if rank == 0 and also:
        line["also"] = {}
        for nm in also:
            if nm == "c4slab":
                line["also"][nm] = slab
                continue
            if nm in ("datagen", "paper_ju", "train", "block", "mv512"):
                try:
                    fn = {"datagen": datagen_budget, "paper_ju": paper_ju_budget, "train": train_budget,
                          "block": block_budget, "mv512": mv_converged_budget}[nm]
                    line["also"][nm] = fn(local, args)
                except Exception as e:  # reported, not hidden
                    line["also"][nm] = {"error": repr(e)}
                continue
            try:
                line["also"][nm] = fixed_budget(nm, local, args, ws, rank)
            except Exception as e:  # reported, not hidden
                line["also"][nm] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)


def fixed_budget(name, local, args, ws, rank):
    """Configs whose random-init-net preconditioner stagnates: time a fixed FGMRES
    iteration budget on the full-size problem (per-iteration throughput)."""
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    from paper_2203_11025_b200 import problems
    cfg = config_for(name)
    cols = columns(cfg, ws, rank, 1)
    ctx, arr = problems.gpu_setup(cfg, device=local)
    Bh = np.ascontiguousarray(problems.rhs_block(arr)[cols])
    nb = Bh.shape[0]
    # whole restart cycles: a budget that ends mid-cycle leaves the cycle's remaining inner
    # steps launched as no-ops on frozen columns (their launches would inflate ms/iteration)
    m = cfg["restart"]
    budget = max(m, (args.budget // m) * m)
    kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=budget, rel_tol=1e-6)
    dev = torch.device("cuda", local)
    dB = torch.from_numpy(Bh).to(dev)
    dX = torch.zeros_like(dB)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    ctx.fgmres_device(cfg["precond"], dB.data_ptr(), dX.data_ptr(), nb, kc, want_report=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dX.zero_()
    e0.record(stream)
    rep = ctx.fgmres_device(cfg["precond"], dB.data_ptr(), dX.data_ptr(), nb, kc)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ctx.set_option("split_vcycle", 0)  # serialised half-batches: un-inflated per-launch event times
    ctx.prof_reset()
    ctx.prof_enable(True)
    dX.zero_()
    ctx.fgmres_device(cfg["precond"], dB.data_ptr(), dX.data_ptr(), nb, kc, want_report=False)
    ctx.prof_enable(False)
    ctx.set_option("split_vcycle", 1)
    torch.cuda.synchronize()
    prof = ctx.prof()
    conv = prof.get("conv3x3", {})
    its = max(1, max(rep.iterations))
    out = {"grid": cfg["n"], "rhs": nb, "precond": cfg["precond"], "iterations_budget": budget, "ms": ms,
           "ms_per_iteration": ms / its,
           "rel_residual_end": [round(float(h[-1] / h[0]), 6) for h in rep.residual_history],
           "converged": [bool(c) for c in rep.converged]}
    if conv.get("ms", 0) > 0:
        out["conv_tflops"] = conv["flops"] / (conv["ms"] / 1e3) / 1e12
        out["conv_share"] = conv["ms"] / max(1e-9, sum(v["ms"] for v in prof.values()))
        # 3xTF32: the tensor pipe executes 3x the useful flops (A_hi [W_hi|W_lo] + A_lo W_hi)
        tp, tsrc = tf32_peak()
        out["conv_tensor_pipe_frac"] = 3.0 * out["conv_tflops"] / tp
        out["conv_tensor_peak"] = {"tflops": tp, "source": tsrc}
        # the 16-channel layers are HBM-bound even at 3x the flops (108 issued flop/B against
        # a machine balance of ~170): the bound of the conv class is the larger of its
        # activation traffic at the HBM peak and its issued flops at the tensor peak
        hbm = peaks()[0].get("hbm_gbs", 6650.0)
        t_hbm = conv["bytes"] / (hbm * 1e9)
        t_tc = 3.0 * conv["flops"] / (tp * 1e12)
        out["conv_hbm_frac"] = t_hbm / (conv["ms"] / 1e3)
        out["conv_roofline_frac"] = max(t_hbm, t_tc) / (conv["ms"] / 1e3)
    # per kernel class: achieved GB/s (algorithmic bytes) and fraction of
    # the measured HBM peak -- meaningful here, the working sets exceed L2 from c2 on
    pk, _ = peaks()
    total = max(1e-9, sum(v["ms"] for v in prof.values()))
    pcls = [k for k in ("vcycle_down", "vcycle_up", "coarse_solve", "smooth", "transfer") if prof.get(k, {}).get("launches")]
    pc_ms = sum(prof[k]["ms"] for k in pcls)
    pc_bytes = sum(prof[k]["bytes"] for k in pcls)
    if pc_ms > 0:
        out["vcycle_apply"] = {"classes": pcls, "gbs": pc_bytes / (pc_ms / 1e3) / 1e9,
                               "hbm_frac": pc_bytes / (pc_ms / 1e3) / 1e9 / pk.get("hbm_gbs", 6650.0),
                               "ms_per_iteration": pc_ms / its}
    out["kernels"] = {}
    for k, v in prof.items():
        if not v["launches"]:
            continue
        row = {"ms_per_iteration": v["ms"] / its, "share": v["ms"] / total}
        if v["bytes"] > 0:
            row["gbs"] = v["bytes"] / (v["ms"] / 1e3) / 1e9
            row["hbm_frac"] = row["gbs"] / pk.get("hbm_gbs", 6650.0)
        if v["flops"] > 0:
            row["tflops"] = v["flops"] / (v["ms"] / 1e3) / 1e12
        out["kernels"][k] = row
    ctx.close()
    if rank == 0 and not args.no_cpu:
        try:
            cr = cpu_reference_budget(name, CPU_BUDGET.get(name, 1))
            cr["speedup_per_iteration_per_rhs"] = (cr["ms_per_iteration"] / (out["ms_per_iteration"] / nb))
            out["cpu_reference"] = cr
        except Exception as e:  # reported, not hidden
            out["cpu_reference"] = {"error": repr(e)}
    return out


# FGMRES iterations of the CPU reference per `also` config (bounded: ~1-15 s each)
CPU_BUDGET = {"c1": 3, "c2": 1, "c3": 1, "c4": 1}


def datagen_budget(local, args):
    """Training pairs (gen_sample_pair, inc/datagen.hpp:191-219)
    on the c0 problem through the public C ABI (host draws, per-k batched
    FGMRES(M_V) on the device, r / e back in host memory): pairs/s, against
    the reference's own gen_sample_pair on one host thread."""
    import time
    import torch
    from paper_2203_11025_b200 import problems
    cfg = config_for("c0")
    ctx, arr = problems.gpu_setup(cfg, device=local)
    count = 2 * torch.cuda.get_device_properties(local).multi_processor_count
    seeds = np.arange(1000, 1000 + count, dtype=np.uint64)
    ctx.gen_sample_pairs(seeds[:16])  # warm-up: graphs / buffers
    dev = torch.device("cuda", local)
    st = torch.cuda.ExternalStream(ctx.stream, device=dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r, e, k = ctx.gen_sample_pairs(seeds)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out = {"grid": cfg["n"], "pairs": int(count), "k_mean": float(k.mean()), "ms": ms,
           "pairs_per_s": count / (ms / 1e3), "path": "hb_gen_sample_pairs (host draws + device FGMRES, host r/e)"}
    ctx.close()
    try:  # the reference's gen_sample_pair, one host thread, bounded sample
        from oracle import oracle as O
        if O.have_ref():
            H = O.RefHierarchy(arr["kappa2"], arr["gamma"], arr["omega"], arr["lo"], arr["hi"], levels=cfg["levels"])
            t0, n = time.perf_counter(), 0
            while time.perf_counter() - t0 < 3.0:
                O.ref_gen_sample_pair(H, 1000 + n, -1, 10)
                n += 1
            dt = time.perf_counter() - t0
            out["cpu_reference"] = {"pairs_per_s": n / dt, "pairs": n, "cores": 1, "kind": "reference"}
    except Exception as ex:  # reported, not hidden
        out["cpu_reference"] = {"error": repr(ex)}
    return out


def mv_converged_budget(local, args, name="c2"):
    """A CONVERGED solve at scale: M_V (3-level SL V-cycle, GMRES(10) coarsest;
    no network, so it reaches 1e-6) FGMRES(20) on config `name`'s grid, medium
    and RHS block, every column to 1e-6.  Device time of the whole solve (RHS
    resident), solves/s; beside it the reference's CPU cost per FGMRES
    iteration of one column on one host core (oracle/_ref, 5 iterations) times
    the device's iteration count (extrapolated, labelled)."""
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    from paper_2203_11025_b200 import problems
    cfg = dict(config_for(name))
    cfg.update(precond="v", net=None, enc=None, coarse="gmres", coarse_iters=10, restart=20, levels=3)
    ctx, arr = problems.gpu_setup(cfg, device=local)
    Bh = np.ascontiguousarray(problems.rhs_block(arr))
    nb = Bh.shape[0]
    kc = hg.KrylovConfig(restart=20, max_iters=4000, rel_tol=1e-6)
    dev = torch.device("cuda", local)
    dB = torch.from_numpy(Bh).to(dev)
    dX = torch.zeros_like(dB)
    st = torch.cuda.ExternalStream(ctx.stream, device=dev)
    ctx.fgmres_device("v", dB.data_ptr(), dX.data_ptr(), nb, hg.KrylovConfig(restart=20, max_iters=40), want_report=False)
    torch.cuda.synchronize()
    dX.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    rep = ctx.fgmres_device("v", dB.data_ptr(), dX.data_ptr(), nb, kc)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    its = int(max(rep.iterations))
    out = {"grid": cfg["n"], "rhs": nb, "precond": "M_V (3 levels, GMRES(10) coarsest)", "restart": 20,
           "iterations_max": its, "iterations_min": int(min(rep.iterations)), "all_converged": bool(all(rep.converged)),
           "ms": ms, "solves_per_s": nb / (ms / 1e3)}
    ctx.close()
    if not args.no_cpu:
        try:
            from oracle import oracle as O
            from oracle import problems as OP
            acfg = ref_config(name)
            acfg.update(precond="v", net=None, enc=None, coarse="gmres", coarse_iters=10, restart=20, levels=3)
            a2 = OP.problem_arrays(acfg)
            kind = "reference" if O.have_ref() else "port"
            H, P = ref_preconditioner(O, kind, acfg, a2)
            solve = O.ref_fgmres if kind == "reference" else O.fgmres
            t0 = time.perf_counter()
            solve(P, OP.rhs_block(a2)[:1], restart=20, max_iters=5, nthreads=1)
            per_it = (time.perf_counter() - t0) / 5
            out["cpu_reference"] = {"kind": kind, "cores": 1, "cpu": cpu_model(), "ms_per_iteration": 1e3 * per_it,
                                    "extrapolated_solve_s_per_rhs": per_it * its,
                                    "extrapolation": f"EXTRAPOLATED: 5 measured iterations x the device's {its} "
                                                     "iterations, assuming the reference needs the same count "
                                                     "(shown +-1 for M_V at 256^2 / 512^2 on the c0 medium, "
                                                     "tests/test_scale_parity.py)",
                                    "speedup_solves_per_s": (nb / (ms / 1e3)) / (1.0 / (per_it * its))}
            del H, P
        except Exception as ex:  # reported, not hidden
            out["cpu_reference"] = {"error": repr(ex)}
    return out


def block_budget(local, args):
    """True block FGMRES (hb_block_fgmres, PAPER.md:580
    block-size study) on the c0 problem: 8 seeded complex-normal right-hand
    sides solved as ONE block Krylov space vs the same 8 as independent
    columns (block_fgmres semantics), M_V, restart 10, to 1e-6.  Device time
    of the whole solve (host c128 I/O included in both)."""
    import time
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    from paper_2203_11025_b200 import problems
    cfg = config_for("c0")
    ctx, arr = problems.gpu_setup(cfg, device=local)
    p = 8
    rng = np.random.default_rng(11)
    B = rng.standard_normal((p, cfg["n"], cfg["n"])) + 1j * rng.standard_normal((p, cfg["n"], cfg["n"]))
    kc = hg.KrylovConfig(restart=10, max_iters=400, rel_tol=1e-6)
    out = {"grid": cfg["n"], "rhs": p, "restart": 10}
    for name, fn in (("block", ctx.block_fgmres), ("columns", ctx.fgmres)):
        fn("v", B, kc)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        X, rep = fn("v", B, kc)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[name] = {"iterations": int(max(rep.iterations)), "converged": bool(all(rep.converged)),
                     "ms": 1e3 * dt, "solves_per_s": p / dt,
                     "preconditioner_applies": int(max(rep.iterations)) * p}
    ctx.close()
    return out


def paper_ju_budget(local, args):
    """M_JU with the paper's U-Net (inc/precond.hpp:104-139, UNetConfig defaults
    inc/unet.hpp:113-120: 3 levels, base 16, 1 ResNet per level, 3 bottleneck
    ResNets, 5x5 up/down) on the c0 problem, NetworkWeights default init with
    the batch-norm buffers marked initialised (mark_bn_initialized): applies/s
    for a batch of 16 and the conv rate."""
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    from paper_2203_11025_b200 import problems
    cfg = config_for("c0")
    ctx, arr = problems.gpu_setup(cfg, device=local)
    ctx.set_paper_net(hg.UNetConfig(), "standalone")
    for name, dims in ctx.paper_params():
        if name.endswith(".count"):
            ctx.paper_param(name, np.ones(dims, np.float32))
    B = 16
    n = cfg["n"]
    r = np.random.default_rng(0).standard_normal((B, n, n)) + 1j * np.random.default_rng(1).standard_normal((B, n, n))
    out = {"grid": n, "net": "UNetConfig() standalone (3 levels, base 16)"}
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    for B in (16, 128):
        r = np.random.default_rng(0).standard_normal((B, n, n)) + 1j * np.random.default_rng(1).standard_normal((B, n, n))
        dr = torch.from_numpy(r.astype(np.complex64)).to(f"cuda:{local}")
        dz = torch.zeros_like(dr)
        ctx.precond_apply_device("ju", dr.data_ptr(), dz.data_ptr(), B)
        torch.cuda.synchronize()
        # whole applies back to back on the library stream (launch gaps included)
        reps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            ctx.precond_apply_device("ju", dr.data_ptr(), dz.data_ptr(), B)
        e1.record(stream)
        torch.cuda.synchronize()
        app_ms = e0.elapsed_time(e1) / reps
        # per kernel class (eager, events per launch): the conv rate
        ctx.prof_reset()
        ctx.prof_enable(True)
        for _ in range(3):
            ctx.precond_apply_device("ju", dr.data_ptr(), dz.data_ptr(), B)
        ctx.prof_enable(False)
        prof = ctx.prof()
        cls_ms = sum(v["ms"] for v in prof.values())
        conv = prof.get("conv3x3", {})
        row = {"us_per_apply_batch": 1e3 * app_ms, "applies_per_s": B / (app_ms / 1e3),
               "conv_share": conv.get("ms", 0) / max(1e-9, cls_ms),
               "conv_tflops": conv["flops"] / (conv["ms"] / 1e3) / 1e12 if conv.get("ms") else None}
        if B == 16:
            out.update(batch=B, **row)
        else:
            out[f"batch{B}"] = row
    out["note"] = ("hb_precond_apply_device on device c64 fields: CUDA events around back-to-back whole applies "
                   "(launch gaps included); conv rate from the per-class event pass")
    ctx.close()
    return out


def train_budget(local, args):
    """Training of the paper U-Net: one run_batch (train-
    mode forward, MSE, reverse sweep) + adam_step per step, UNetConfig()
    defaults at 128^2 with the paper's retraining batch of 20, through the C
    ABI (host batch in, host loss / output / weights back every step); against
    the reference's own run_batch + adam_step on one host thread (one batch)."""
    import time
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    n, B, steps = 128, 20, 10
    rs = np.random.default_rng(0)
    x = rs.standard_normal((B, 4, n, n)).astype(np.float32)
    x[:, :2] *= 1e-3
    t = rs.standard_normal((B, 2, n, n)).astype(np.float32)
    ctx = hg.Context(local)
    ctx.set_paper_net(hg.UNetConfig(), "standalone")
    ctx.paper_init(3)
    for _ in range(2):
        ctx.paper_train_batch(x, t, step=True, lr=1e-5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        loss, _ = ctx.paper_train_batch(x, t, step=True, lr=1e-5)
    dt = (time.perf_counter() - t0) / steps
    out = {"grid": n, "batch": B, "net": "UNetConfig() standalone (3 levels, base 16)", "ms_per_batch": dt * 1e3,
           "samples_per_s": B / dt, "loss": loss,
           "path": "hb_paper_train_batch (host batch in; loss, output and weights back each step)"}
    ctx.close()
    try:
        from oracle import oracle as O
        if O.have_ref():
            net = O.RefPaperNet(levels=3, base=16, rpl=1, bot=3, kud=5, kres=3, variant=0, seed=3)
            t0 = time.perf_counter()
            net.train_batch(x, t, step=True, lr=1e-5)
            dr = time.perf_counter() - t0
            out["cpu_reference"] = {"ms_per_batch": dr * 1e3, "samples_per_s": B / dr, "cores": 1, "kind": "reference"}
    except Exception as ex:  # reported, not hidden
        out["cpu_reference"] = {"error": repr(ex)}
    return out


SLAB_DEADLINE_S = 240.0  # c4slab over NCCL: setup (~20 s) + three fixed budgets (< 1 s) with a wide margin


def run_with_deadline(fn, local, seconds):
    """fn() on a worker thread bound to this rank's GPU; (result, False), or
    ({"error": ...}, True) when it has not returned within `seconds` (None: no
    deadline, run inline).  Exceptions are reported in the result, not hidden."""
    def guarded():
        try:
            return fn()
        except Exception as e:
            return {"error": repr(e)}
    if seconds is None:
        return guarded(), False
    import threading
    box = {}

    def work():
        try:
            import torch
            if torch.cuda.is_available():
                torch.cuda.set_device(local)
        except Exception:
            pass
        box["out"] = guarded()
    th = threading.Thread(target=work, daemon=True)
    th.start()
    th.join(seconds)
    if th.is_alive():
        return {"error": f"no result within {seconds:.0f} s (collective wedged?); entry skipped"}, True
    return box["out"], False


def slab_budget(local, args, ws, rank):
    """c4 (one 4096^2 RHS, 4-level V-cycle, U-Net coarsest at 512^2) on row slabs
    (SURVEY 8(e)): one slab per rank over NCCL when ws > 1, else an in-process
    group of 2 slabs on this GPU (device-copy halos: the decomposition's
    overhead against the whole-grid c4 entry).  Marginal device time per FGMRES
    iteration = difference of two fixed budgets (same I/O and setup), max over
    ranks."""
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    from paper_2203_11025_b200 import problems
    cfg = config_for("c4")
    arr = problems.problem_arrays(cfg)
    if ws == 1:
        ctxs = [problems.gpu_setup(cfg, device=local, arr=arr)[0] for _ in range(2)]
        hg.slab_init_local(ctxs)
        lead, nslabs, transport = ctxs[0], 2, "in-process (device copies), 1 GPU"
    else:
        lead = problems.gpu_setup(cfg, device=local, arr=arr)[0]
        hg.slab_init_distributed(lead)
        ctxs, nslabs, transport = [lead], ws, "nccl"
    lo, hi = lead.slab_rows()
    B = np.ascontiguousarray(problems.rhs_block(arr)[:, lo:hi])
    dev = torch.device("cuda", local)
    st = torch.cuda.ExternalStream(lead.stream, device=dev)

    def run(budget):
        kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=budget, rel_tol=1e-6)
        barrier(ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        X, rep = lead.fgmres_slab(cfg["precond"], B, kc)
        e1.record(st)
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1), ws), rep

    b1, b2 = 10, 10 + args.budget
    run(b1)  # warm-up: allocations, graph capture
    t1, _ = run(b1)
    t2, rep = run(b2)
    out = {"grid": cfg["n"], "levels": cfg["levels"], "slabs": nslabs, "transport": transport,
           "rows_per_slab": hi - lo if ws > 1 else cfg["n"] // 2,
           "ms_per_iteration": (t2 - t1) / (b2 - b1), "iterations": [b1, b2],
           "rel_residual_end": round(float(rep.residual_history[0][-1] / rep.residual_history[0][0]), 6),
           "note": "coarsest level all-gathered and solved replicated (NCCL ranks: every rank; in-process group on one GPU: once, solution copied to the other slabs); 2 ghost rows per slab level"}
    for c in ctxs:
        c.close()
    return out


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: start N ranks of this script (one per
    GPU, LOCAL_RANK = i) with torchrun's environment, rank 0's stdout is the JSON
    line.  NCCL's init log stays on (NCCL_DEBUG=INFO on stderr) so the ranks are
    visible."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for i in range(n):
        env = dict(os.environ, WORLD_SIZE=str(n), RANK=str(i), LOCAL_RANK=str(i), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if i == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def dry_run(args, ws, rank):
    """Host plumbing only (CPU, gloo): rank -> column partition, barriers,
    max-over-ranks timing and the solve count -- used by the CPU test of the
    self-launch path.  Prints a line marked dry_run (not a measurement)."""
    cfg = ref_config(args.config)
    cols = columns(cfg, ws, rank, args.replicas or 3)
    barrier(ws)
    t = max_over_ranks(1.0 + rank, ws)
    solves = sum_over_ranks(len(cols), ws)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "config": {"workload": args.config}, "rhs_total": solves,
                          "rank0_columns": cols, "max_over_ranks": t}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c0")
    ap.add_argument("--replicas", type=int, default=0, help="solves per GPU per step for single-RHS configs "
                                                              "(0 = 6 per SM: two per SM in each of the 3 column groups)")
    ap.add_argument("--also", default="datagen,c1,c2,c3,c4,c4slab,mv512,paper_ju,train,block", help="comma list of configs measured on a fixed iteration budget "
                                                       "(rounded down to whole restart cycles, at least one)")
    ap.add_argument("--budget", type=int, default=20)
    ap.add_argument("--opt", action="append", default=[], help="library option key=value (hb_set_option)")
    ap.add_argument("--groups", type=int, default=3, help="independent column groups (solver contexts on their own "
                                                          "streams and host threads) per GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pipeline", dest="no_pipeline", action="store_true",
                    help="e2e: only the per-step-joined measurement")
    ap.add_argument("--dry-run", action="store_true", help="host plumbing only (no GPU work; CPU test of --gpus N)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(spawn_ranks(args.gpus))
    ws, rank, local = dist_init()
    if args.dry_run:
        dry_run(args, ws, rank)
    elif args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        if ws != args.gpus and rank == 0:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {ws}; measuring {ws} GPU(s)", file=sys.stderr)
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
