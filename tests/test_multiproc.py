"""World-size-2 tests of the multi-GPU host path on CPU (gloo).

The B200 path shards the independent right-hand sides of c1-c3 across ranks
and runs replicas of the single-RHS c0: no data-path
collective, only the bench's barrier and max-over-ranks timing reduction.
These tests run that host logic with two gloo ranks: the rank -> column
partition (bench.columns), the timing reduction (bench.max_over_ranks), and a
sharded block solve whose per-rank results, gathered, equal the single-process
block solve bit for bit (columns are independent Arnoldi processes,
inc/krylov.hpp:78-82; the oracle stands in for the per-rank device solve).
"""
import math
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n=32, B=4):
    from oracle import oracle as O
    om = 2 * math.pi * 1.5 * n / 10
    k2 = O.make_medium(n, n, 77)
    g = O.absorbing_layer(n, n, 4, 2 * om)
    rhs = O.random_complex_normal(131, (B, n, n))
    return k2, g, om, rhs


def _rank_main(rank, ws, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import bench
    from oracle import oracle as O
    w, r, _ = bench.dist_init()
    assert (w, r) == (ws, rank) and dist.get_backend() == "gloo"
    # c1 (B = 8 point sources) sharded over the ranks; c0 (B = 1) replicated
    cols = {name: bench.columns(bench.config_for(name), ws, rank, 3) for name in ("c0", "c1", "c2")}
    # sharded M_V block solve (the oracle stands in for the per-rank device solve)
    k2, g, om, rhs = _problem()
    mine = bench.columns({"B": rhs.shape[0]}, ws, rank, 1)
    H = O.Hierarchy(k2, g, om, 1 / 16, 1 / 2.25, levels=2)
    X, rep = O.fgmres(O.Precond("v", H), rhs[mine], max_iters=120)
    # timing reduction used by bench.py: max over ranks
    tmax = bench.max_over_ranks(1.0 + rank, ws)
    bench.barrier(ws)
    parts = [None] * ws
    dist.all_gather_object(parts, {"rank": rank, "cols": cols, "mine": mine, "X": X, "hist": rep["history"],
                                   "tmax": tmax})
    if rank == 0:
        np.save(os.path.join(out_dir, "parts.npy"), np.array(parts, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_rhs_sharding_gloo(tmp_path):
    import torch.multiprocessing as mp
    ws = 2
    mp.start_processes(_rank_main, args=(ws, _free_port(), str(tmp_path)), nprocs=ws, start_method="spawn")
    parts = list(np.load(tmp_path / "parts.npy", allow_pickle=True))
    assert [p["rank"] for p in parts] == [0, 1]
    # partition: c1 / c2 columns disjoint and complete; c0 replicated per rank
    for name, B in (("c1", 8), ("c2", 16)):
        got = sorted(c for p in parts for c in p["cols"][name])
        assert got == list(range(B))
    assert all(p["cols"]["c0"] == [0, 0, 0] for p in parts)
    # the timing reduction is a max over ranks
    assert all(p["tmax"] == 2.0 for p in parts)
    # gathered sharded solve == single-process block solve, bit for bit
    from oracle import oracle as O
    k2, g, om, rhs = _problem()
    H = O.Hierarchy(k2, g, om, 1 / 16, 1 / 2.25, levels=2)
    X, rep = O.fgmres(O.Precond("v", H), rhs, max_iters=120)
    for p in parts:
        for i, c in enumerate(p["mine"]):
            assert np.array_equal(p["X"][i], X[c])
            assert np.array_equal(p["hist"][i], rep["history"][c])


@pytest.mark.timeout(600)
def test_bench_gpus_flag_self_launches_ranks():
    """`bench.py --gpus N` without torchrun starts N ranks itself (here: 2 gloo
    ranks on CPU, host plumbing only) and rank 0 reports n_gpus = N with the
    RHS block sharded over the ranks (uneven world sizes included)."""
    import json
    import subprocess
    for n, cfg, B in ((2, "c1", 8), (3, "c2", 16)):
        env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dry-run",
                            "--config", cfg], capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        line = json.loads(r.stdout.strip().splitlines()[-1])
        assert line["dry_run"] and line["n_gpus"] == n
        assert line["rhs_total"] == B and line["max_over_ranks"] == float(n)
        assert line["rank0_columns"] == list(range(-(-B // n)))


def test_bench_deadline_guard_reports_instead_of_hanging():
    """bench.run_with_deadline: the NCCL slab entry runs under a deadline so a
    wedged collective cannot take the headline line with it; results and
    exceptions pass through, a late worker is reported as such."""
    import time

    sys.path.insert(0, ROOT)
    import bench

    assert bench.run_with_deadline(lambda: {"ok": 1}, 0, None) == ({"ok": 1}, False)
    assert bench.run_with_deadline(lambda: {"ok": 2}, 0, 5.0) == ({"ok": 2}, False)
    out, wedged = bench.run_with_deadline(lambda: 1 / 0, 0, 5.0)
    assert not wedged and "ZeroDivisionError" in out["error"]
    out, wedged = bench.run_with_deadline(lambda: time.sleep(3.0), 0, 0.2)
    assert wedged and "no result within" in out["error"]
