#!/usr/bin/env python3
"""Runs BASELINE.json's single-GPU configurations C1-C4 end to end on the GPU
(the reference mapping of SURVEY.md 8(d) / DESIGN.md section 2) and, beside
each, the reference's own CPU solver (oracle/_ref) on a bounded sample.
Prints one JSON object per config; `--out FILE` also writes them as a list.

  python configs.py [--only c1,c2,c3,c4] [--out profiles/r1_configs.json]
  python configs.py --only c5 [--c5-ranks 0,3,7] [--c5-iters 200]

C5 (n = 2^32, 8 GPUs) cannot run whole on the single GPU available here: the
c5 entry builds the row-block shard of each requested rank of the 8-way split
(the generator draws sigma / the fill on the device with mt19937_64
jump-ahead, so a rank never replays or stores the 2^32-entry streams) and times
that rank's own launches (two-iteration kernel + finalise) on the one GPU.
The halo stores and the 8-double all-reduce of the real 8-GPU run are not in
these numbers (no neighbours exist), so the rate is a per-rank compute figure.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

THETA = 2 * math.pi / 10


def log_sigma(n):
    return [math.pow(10.0, float(i) / float(n - 1)) for i in range(n)]


CONFIGS = {
    "c1": dict(desc="FISTA, n=2^12 x m=2^13, log-spaced sigma (kappa=100), s=n/100, seed 0, to the 1e-8 gap",
               gen=dict(n=1 << 12, stages=1, s_divisor=100, seed=0), sigma="log", solver="fista",
               rel_gap=1e-8, max_iters=100000),
    "c2": dict(desc="block PCDM (B=256), n=2^15 x m=2^16, q=1, s=n/100, seed 1, 100 epochs",
               gen=dict(n=1 << 15, stages=1, q=1, s_divisor=100, seed=1), solver="pcdm",
               max_iters=100, block=256, solver_seed=1),
    "c3": dict(desc="pdNCG, n=2^19 x m=2^20, q=2, s=n/1000, seed 2, mu=1e-5 fixed, 30 Newton steps",
               gen=dict(n=1 << 19, stages=1, q=2, s_divisor=1000, seed=2), solver="newton_cg",
               max_iters=30),
    "c4": dict(desc="FISTA, n=2^27 x m=2^28, 4 stages, q=1, s=n/1000, seed 3, 500 iterations",
               gen=dict(n=1 << 27, stages=4, q=1, s_divisor=1000, seed=3), solver="fista",
               max_iters=500),
}

# CPU runs of the reference (oracle/_ref): the whole configuration (None) or,
# for C4 (~8 s per iteration on one core: 500 iterations would be ~70 min),
# (n, iterations) at the configuration's own n, extrapolated in the iteration
# count only ("10 iterations, extrapolated and labelled")
CPU_SAMPLE = {"c1": None, "c2": None, "c3": None, "c4": (1 << 27, 10)}


def run_gpu(name, c):
    import torch

    from paper_1503_03520_b200 import l1bench

    kw = dict(c["gen"], theta=THETA)
    if c.get("sigma") == "log":
        kw["sigma"] = log_sigma(kw["n"])
    t0 = time.perf_counter()
    inst = l1bench.build_instance(lazy_sparse=(c["solver"] == "fista"), **kw)
    gen_s = time.perf_counter() - t0
    f_star = inst.objective_at_planted()
    b = inst.b
    f0 = 0.5 * float((b * b).sum())
    target = None
    if "rel_gap" in c:
        target = f_star + c["rel_gap"] * max(f0 - f_star, 0.0)
    cfg = l1bench.SolverConfig(id=c["solver"], max_iters=c["max_iters"], target_objective=target,
                               block=c.get("block", 256), seed=c.get("solver_seed", 0),
                               max_seconds=3600.0)
    if c["solver"] != "fista" or inst.n < (1 << 20):  # warm-up run (one-time library set-up)
        l1bench.run_solver(inst, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = l1bench.run_solver(inst, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"config": name, "desc": c["desc"], "n": inst.n, "m": inst.m, "generate_s": gen_s,
           "solver": c["solver"], "status": str(tr.status), "iterations": tr.iterations,
           "solve_wall_s": wall, "solve_device_s": tr.elapsed_s, "f_final": tr.final_objective,
           "f_star": f_star, "rel_gap_final": (tr.final_objective - f_star) / max(f0 - f_star, 1e-300),
           "matvecs": tr.total_matvecs}
    if c["solver"] == "newton_cg":
        out["pcg_iterations"] = tr.total_pcg_iterations
        out["smoothing_band_tau_n_mu"] = inst.tau * inst.n * 1e-5
    if target is not None:
        out["target"] = target
        out["time_to_target_s"] = tr.time_to_target
    if tr.iterations:
        out["iters_per_s"] = tr.iterations / max(tr.elapsed_s, 1e-12)
    if c["solver"] == "fista" and inst.n > (1 << 20):
        # the contracted arithmetic (bench.py's headline; <= 1e-12 of these iterates) beside the
        # bit-identical run above
        from dataclasses import replace

        trf = l1bench.run_solver(inst, replace(cfg, arith="fma"))
        out["arith"] = "exact"
        out["arith_fma"] = {"iterations": trf.iterations, "solve_device_s": trf.elapsed_s,
                            "iters_per_s": trf.iterations / max(trf.elapsed_s, 1e-12),
                            "f_final": trf.final_objective,
                            "rel_df_vs_exact": abs(trf.final_objective - tr.final_objective) / abs(tr.final_objective)}
    if c["solver"] == "pcdm":
        # the reference's own algorithm on the same instance: serial CD (solvers.cpp:414-482),
        # bit-exact with the reference, same epoch budget -- the like-for-like rate beside cpu_reference
        scfg = l1bench.SolverConfig(id="cd", max_iters=c["max_iters"], seed=c.get("solver_seed", 0),
                                    max_seconds=3600.0)
        l1bench.run_solver(inst, scfg)
        trc = l1bench.run_solver(inst, scfg)
        out["serial_cd"] = {"epochs": trc.iterations, "solve_device_s": trc.elapsed_s,
                            "epochs_per_s": trc.iterations / max(trc.elapsed_s, 1e-12),
                            "f_final": trc.final_objective}
    return out


def run_cpu(name, c):
    from pyoracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        return {"unavailable": "oracle/_ref/libl1ref.so not built"}
    ref = Reference()
    kw = dict(c["gen"], theta=THETA)
    sample = CPU_SAMPLE[name]
    iters = c["max_iters"]
    if sample:
        kw["n"], iters = sample
    if c.get("sigma") == "log":
        import numpy as np

        kw["sigma"] = np.array(log_sigma(kw["n"]))
    inst = ref.build_instance(**kw)
    f0 = 0.5 * float((inst.b() ** 2).sum())
    target = None
    if "rel_gap" in c:
        target = inst.f_star + c["rel_gap"] * max(f0 - inst.f_star, 0.0)
    solver = "cd" if c["solver"] == "pcdm" else c["solver"]
    t0 = time.perf_counter()
    tr, _ = inst.solve(solver, max_iters=iters, target=target, varpi=c.get("block", 1),
                       seed=c.get("solver_seed", 0))
    wall = time.perf_counter() - t0
    n_iter = int(tr["iter"][-1]) if len(tr["iter"]) else 0
    out = {"kind": "reference", "cores": 1, "n": inst.n, "solver": solver, "iterations": n_iter,
           "wall_s": wall, "f_final": tr["final_objective"],
           "sample": "full run" if not sample else
           f"n={kw['n']} (the config's own n), {iters} of the config's {c['max_iters']} iterations"}
    if n_iter:
        out["iters_per_s"] = n_iter / max(tr["elapsed_s_total"], 1e-12)
        out["solve_s"] = float(tr["elapsed_s_total"])
        if sample:
            out["solve_s_extrapolated_to_config_iterations"] = c["max_iters"] / out["iters_per_s"]
    if target is not None:
        out["time_to_target_s"] = float(tr["elapsed_s"][-1])
    return out


C5 = dict(n=1 << 32, stages=4, q=0, s_divisor=10000, seed=4, theta=THETA)


def run_c5(ranks, iters, world=8, arith="fma"):
    """Per-rank shards of C5 on the one GPU (see the module docstring)."""
    import gc

    import torch

    from paper_1503_03520_b200 import l1bench
    from paper_1503_03520_b200.distributed import CudaShard

    out = {"config": "c5", "desc": "FISTA, n=2^32 x m=2^33, 4 stages, q=0, s=n/10000, seed 4; "
                                   f"rank shards of the {world}-way row split, one at a time on one GPU",
           "world": world, "iterations_timed": iters, "arith": arith, "ranks": []}
    for r in ranks:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sh = CudaShard(C5, r, world, 0, l1bench.SolverConfig(max_iters=iters + 8, op="matrix_free", arith=arith))
        torch.cuda.synchronize()
        gen_s = time.perf_counter() - t0
        assert sh.single and sh.pairs, "C5 shards run the two-iteration kernel"
        sh.finalize()  # f_0 from this rank's ||b_own||^2 (no all-reduce: one rank here)
        for _ in range(2):
            sh.k1()
            sh.finalize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(iters // 2):
            sh.k1()
            sh.finalize()
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / (iters // 2 * 2)
        info = sh.inst.info
        out["ranks"].append({"rank": r, "rows": [int(info.row_begin), int(info.row_end)],
                             "generate_s": gen_s, "ms_per_iteration": ms,
                             "device_gb": int(info.device_bytes) / 1e9,
                             "gbs_algorithmic": 24 * sh.own / (ms * 1e-3) / 1e9})
        print(json.dumps(out["ranks"][-1]), flush=True)
        del sh
        gc.collect()
        torch.cuda.empty_cache()
    worst = max(x["ms_per_iteration"] for x in out["ranks"])
    out["max_rank_ms_per_iteration"] = worst
    out["projected_iters_per_s_compute_only"] = 1000.0 / worst
    out["note"] = ("per-rank device time of the rank's own launches; the 8-GPU run adds the halo "
                   "stores to the neighbours and one 8-double all-reduce per two iterations")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c3,c4")
    ap.add_argument("--c5-ranks", default="0,3,7")
    ap.add_argument("--c5-iters", type=int, default=200)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    res = []
    for name in args.only.split(","):
        if name == "c5":
            r = run_c5([int(x) for x in args.c5_ranks.split(",")], args.c5_iters)
            print(json.dumps(r), flush=True)
            res.append(r)
            continue
        c = CONFIGS[name]
        r = run_gpu(name, c)
        if not args.no_cpu:
            r["cpu_reference"] = run_cpu(name, c)
        print(json.dumps(r), flush=True)
        res.append(r)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
