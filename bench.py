#!/usr/bin/env python
"""Benchmark: Helmholtz solves/s to 1e-6 relative residual (BASELINE.json metric)
through the B200 FGMRES + SL-multigrid (+ U-Net) hot path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c0]

Workload: the headline line is config c0 --
the only BASELINE config whose solve reaches 1e-6 with seeded random-init
weights (configs c1-c4 put a random-init U-Net in the preconditioner and
stagnate; the oracle shows it).  One step = one FGMRES(10) solve of the c0
problem (128^2, M_V 3 levels, GMRES(10) coarsest) to 1e-6, inputs resident in
HBM.  L2 is flushed (a 512 MiB write) between timed steps.  c1 (the U-Net
coarse-solver config) is measured on a fixed iteration budget and reported
under "also".  Multi-GPU: independent replicas / RHS shards, no collective.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Helmholtz solves/s to 1e-6 rel residual"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


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
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
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
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- workloads
def config_for(name):
    from paper_2203_11025_b200 import configs
    return dict(configs.CONFIGS[name])


def shard(cfg, ws, rank):
    """RHS sharding: rank r gets columns [r*B/ws, (r+1)*B/ws); c0/c4: replicas."""
    B = cfg["B"]
    if B >= ws and B % ws == 0 and B > 1:
        return list(range(rank * B // ws, (rank + 1) * B // ws))
    return list(range(B))  # replicas


def cpu_baseline_sample(cfg_name, cfg):
    """The reference CPU path (oracle/_ref = reference headers compiled in place) on
    a bounded sample, 1 thread; falls back to the C restatement ('port')."""
    from oracle import oracle as O
    from paper_2203_11025_b200 import problems
    arr = problems.problem_arrays(cfg)
    B = problems.rhs_block(arr)[:1]
    kind = "reference" if O.have_ref() else "port"
    mk = (lambda *a, **k: O.RefHierarchy(*a, **k)) if kind == "reference" else (lambda *a, **k: O.Hierarchy(*a, **k))
    H = mk(arr["kappa2"], arr["gamma"], arr["omega"], arr["lo"], arr["hi"], levels=cfg["levels"],
           coarse=cfg["coarse"], coarse_iters=cfg["coarse_iters"])
    P = (O.RefPrecond if kind == "reference" else O.Precond)("v", H)
    t0 = time.perf_counter()
    if kind == "reference":
        X, rep = O.ref_fgmres(P, B, restart=cfg["restart"], max_iters=cfg["max_iters"], nthreads=1)
    else:
        X, rep = O.fgmres(P, B, restart=cfg["restart"], max_iters=cfg["max_iters"], nthreads=1)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": "solves/s", "cores": 1, "kind": kind,
            "sample": f"1 full {cfg_name} solve ({int(rep['iterations'][0])} FGMRES iterations, "
                      f"converged={bool(rep['converged'][0])}), 1 thread, {dt:.3f} s"}


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref) on
    all host threads; replicas of the workload, one per thread."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2203_11025_b200 import problems
    cfg = config_for(args.config)
    arr = problems.problem_arrays(cfg)
    Bfull = problems.rhs_block(arr)
    threads = os.cpu_count() or 1
    kind = "reference" if O.have_ref() else "port"
    mk = O.RefHierarchy if kind == "reference" else O.Hierarchy
    H = mk(arr["kappa2"], arr["gamma"], arr["omega"], arr["lo"], arr["hi"], levels=cfg["levels"],
           coarse=cfg["coarse"], coarse_iters=cfg["coarse_iters"])
    P = (O.RefPrecond if kind == "reference" else O.Precond)("v", H)
    # one column per thread: the workload's RHS, replicated if the config has fewer RHS than threads
    cols = np.stack([Bfull[i % Bfull.shape[0]] for i in range(threads)])
    solve = O.ref_fgmres if kind == "reference" else O.fgmres
    times, conv = [], []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        X, rep = solve(P, cols, restart=cfg["restart"], max_iters=cfg["max_iters"], nthreads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            conv.append(bool(np.all(rep["converged"])))
    total = sum(times)
    value = threads * args.steps / total
    line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (fp64), fp32 network",
            "data": "synthetic (seeded media / point sources, SURVEY 8(d))", "impl": "reference",
            "config": {"workload": args.config, "grid": cfg["n"], "rhs_per_step": threads,
                       "note": "one replica column per host thread"},
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": kind,
                             "sample": f"{threads} concurrent {args.config} solves per step "
                                       f"(all converged: {all(conv)})"},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def flush_l2(buf):
    buf.add_(1.0)  # 512 MiB write >> 126 MB L2


def run_ours(args, ws, rank, local):
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    from paper_2203_11025_b200 import problems
    torch.cuda.set_device(local)
    cfg = config_for(args.config)
    cols = shard(cfg, ws, rank)
    ctx, arr = problems.gpu_setup(cfg, device=local)
    Bh = problems.rhs_block(arr)[cols]
    nb = Bh.shape[0]
    kc = hg.KrylovConfig(restart=cfg["restart"], max_iters=cfg["max_iters"], rel_tol=1e-6)
    kind = cfg["precond"]
    dev = torch.device("cuda", local)
    dB = torch.from_numpy(Bh).to(dev)
    dX = torch.zeros_like(dB)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)

    def step():
        dX.zero_()
        return ctx.fgmres_device(kind, dB.data_ptr(), dX.data_ptr(), nb, kc, want_report=False)

    for _ in range(args.warmup):
        step()
    dX.zero_()
    rep = ctx.fgmres_device(kind, dB.data_ptr(), dX.data_ptr(), nb, kc)
    torch.cuda.synchronize()
    # timed region: K steps, each bracketed by events on the library stream, L2 flushed in between
    barrier(ws)
    torch.cuda.synchronize()
    n0 = ctx.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            dX.zero_()
            torch.cuda.synchronize()
            ev[k][0].record(stream)
            ctx.fgmres_device(kind, dB.data_ptr(), dX.data_ptr(), nb, kc, want_report=False)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    launches = (ctx.launch_count() - n0) // max(1, args.steps)
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    barrier(ws)
    t_ms = max_over_ranks(t_ms, ws)
    solves = nb * args.steps * ws  # every rank solves nb columns per step
    value = solves / (t_ms / 1e3)

    # e2e through the public C ABI with host (pinned) buffers, copies inside the timed region
    Bpin = torch.from_numpy(Bh).pin_memory()
    Xpin = torch.zeros_like(Bpin).pin_memory()
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        ee[k][0].record(stream)
        X, _ = ctx.fgmres(kind, Bpin.numpy(), kc)
        ee[k][1].record(stream)
    torch.cuda.synchronize()
    e_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ee), ws)
    e2e = {"value": solves / (e_ms / 1e3), "unit": "solves/s", "h2d_bytes_per_step": int(Bh.nbytes),
           "d2h_bytes_per_step": int(Bh.nbytes)}

    # roofline pass (same workload, per-kernel-class CUDA events on the library stream)
    ctx.prof_reset()
    ctx.prof_enable(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    ctx.prof_enable(False)
    prof = ctx.prof()
    total_ms = sum(p["ms"] for p in prof.values()) or 1.0
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    pk, src = peaks()
    name, p = dom
    if p["flops"] > 0:
        achieved = p["flops"] / (p["ms"] / 1e3) / 1e12
        peak = pk.get("bf16_tflops", 1590.0) * 0.5
        rl = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
              "traffic": None, "kernel": name,
              "note": f"peak = 0.5 x {src} bf16 burst (provisional TF32 denominator, BASELINE.md 5)"}
    else:
        achieved = p["bytes"] / (p["ms"] / 1e3) / 1e9 if p["ms"] > 0 else 0.0
        peak = pk.get("hbm_gbs", 6650.0)
        rl = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
              "traffic": None, "kernel": name, "note": f"peak = {src} HBM copy bandwidth"}
    rl["share_of_step"] = p["ms"] / total_ms
    rl["avg_launch_us"] = 1e3 * p["ms"] / max(1, p["launches"])
    kernels = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                   "share": v["ms"] / total_ms} for k, v in prof.items() if v["launches"]}

    line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "complex64 (fp64 reductions/Hessenberg/x), fp32 net",
            "data": "synthetic (seeded media / point sources, SURVEY 8(d))",
            "config": {"workload": args.config, "grid": cfg["n"], "rhs_per_gpu": nb, "levels": cfg["levels"],
                       "coarse": f"{cfg['coarse']}({cfg['coarse_iters']})", "restart": cfg["restart"],
                       "precond": kind, "iterations": [int(i) for i in rep.iterations],
                       "converged": [bool(c) for c in rep.converged], "l2": "flushed (512 MiB write) between steps",
                       "parallelism": f"replicas/rhs-shards x{ws}"},
            "roofline": rl, "kernels": kernels, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample(args.config, cfg)
    if rank == 0 and args.also:
        line["also"] = {}
        for name in [s for s in args.also.split(",") if s]:
            try:
                line["also"][name] = fixed_budget(name, local, args, ws, rank)
            except Exception as e:  # report, do not hide
                line["also"][name] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


def fixed_budget(name, local, args, ws, rank):
    """Configs whose random-init-net preconditioner stagnates: time a fixed FGMRES
    iteration budget on the full-size problem (per-iteration throughput)."""
    import torch
    from paper_2203_11025_b200 import helmgpu as hg
    from paper_2203_11025_b200 import problems
    cfg = config_for(name)
    cols = shard(cfg, ws, rank)
    ctx, arr = problems.gpu_setup(cfg, device=local)
    Bh = problems.rhs_block(arr)[cols]
    nb = Bh.shape[0]
    budget = args.budget
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
    ctx.prof_reset()
    ctx.prof_enable(True)
    dX.zero_()
    ctx.fgmres_device(cfg["precond"], dB.data_ptr(), dX.data_ptr(), nb, kc, want_report=False)
    ctx.prof_enable(False)
    prof = ctx.prof()
    conv = prof.get("conv3x3", {})
    out = {"grid": cfg["n"], "rhs": nb, "iterations_budget": budget, "ms": ms,
           "ms_per_iteration": ms / max(1, max(rep.iterations)),
           "rel_residual_end": [float(h[-1] / h[0]) for h in rep.residual_history],
           "converged": [bool(c) for c in rep.converged]}
    if conv.get("ms", 0) > 0:
        out["conv_tflops"] = conv["flops"] / (conv["ms"] / 1e3) / 1e12
        out["conv_share"] = conv["ms"] / max(1e-9, sum(v["ms"] for v in prof.values()))
    ctx.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c0")
    ap.add_argument("--also", default="c1", help="comma list of configs measured on a fixed iteration budget")
    ap.add_argument("--budget", type=int, default=20)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
