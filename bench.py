#!/usr/bin/env python3
"""Benchmark of the B200 l1-least-squares hot path (BASELINE.json metric:
"solver iters/sec and A*x+A^T*r HBM GB/s vs ~8 TB/s roofline, 1/2/4/8 GPUs").

Workload (N=1): configuration C4 of BASELINE.json -- FISTA, fp64, n = 2^27
columns x m = 2^28 rows (SURVEY.md 8(d) tall reading), 4 Givens stages
(nnz(A) = 8n - 16, ~8 nonzeros per column), uniform q=1 spectrum
(kappa ~ 1e4), x* with n/1000 nonzeros, tau = 1, seed 3.  A step is one FISTA
iteration (A^T r + prox/momentum, A x - b + residual momentum) on the device-
resident instance; inputs (~37 GB streamed per iteration) are far larger than
the 126 MB L2, so no flush is needed between iterations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Default K = 500 (the C4 config's iteration budget), W = 4.

The headline path is the matrix-free two-iteration kernel with fused
multiply-adds (--arith fma, the default: iterates within 1e-12 of the
reference's fista_run, same supports); the same kernel with separately rounded
products (bit-identical to the reference) is timed beside it ("other_arith"),
and the north-star CSR/CSC SpMV path on the same instance ("sparse_path").

Under torchrun (N > 1) the C4 instance is row-sharded across the ranks (strong
scaling; NCCL halo exchange + scalar all-reduce per iteration); see DESIGN.md.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C4 = dict(n=1 << 27, m_ratio=2.0, stages=4, q=1, shift=0.1, s_divisor=1000, gamma=10.0, tau=1.0,
          theta=2 * math.pi / 10, seed=3)
C4_ITERS = 500  # the C4 configuration's iteration budget
METRIC = "solver iters/sec (FISTA, C4)"
UNIT = "iter/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons while the GPU is busy."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.rows = []
        self.proc = None
        self.dev = device_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# matrix-free kernels by l1b_session_kernel_mode: (bytes per launch / n, iterations
# per launch, name); every array at its stored width, each element once
MF_KERNELS = {
    4: (48, 2, "fista_rc2 (two FISTA iterations per launch, matrix-free, residuals recomputed): "
               "x_k, x_{k-1}, sigma, b read, x_{k+1}, x_{k+2} written"),
    3: (40, 1, "fista_rc (one FISTA iteration, matrix-free, residuals recomputed): x_k, x_{k-1}, "
               "sigma, b read, x_{k+1} written"),
    2: (64, 1, "fista_iter (one FISTA iteration, matrix-free, stored residuals)"),
}


def kernel_bytes(path, n, m_act, nnz, ptr_bytes, kmode=None):
    """Algorithmic HBM bytes per launch of the FISTA kernels and iterations per launch."""
    if path == "matrix_free":
        per_n, ipl, _ = MF_KERNELS[kmode]
        return per_n * n, 0, ipl
    k1 = 12 * nnz + ptr_bytes * (n + 1) + 8 * m_act + 32 * n      # CSC + r_y gather + x,y r/w
    k2 = 12 * nnz + ptr_bytes * (m_act + 1) + 8 * n + 32 * m_act  # CSR + x gather + b, r_x r/w, r_y w
    return k1, k2, 1


def time_path(inst, op, args, prof_iters=100, arith="exact"):
    """W warm-up iterations, then exactly K timed iterations between CUDA events
    on the library's stream; inside the timed region every launch is also
    bracketed by events on that stream (l1b_session_profile), which gives the
    kernel's average launch duration for the roofline from the same region.
    A longer continuation (prof_iters) keeps the GPU loaded for the nvidia-smi
    clock sampler and gives a second, long-run kernel time."""
    import torch

    from paper_1503_03520_b200 import l1bench

    cfg = l1bench.SolverConfig(max_iters=args.warmup + args.steps + prof_iters + 10, op=op, arith=arith)
    stream = torch.cuda.ExternalStream(inst.stream)
    sess = l1bench.Session(inst, cfg)
    sess.step(args.warmup)
    torch.cuda.synchronize()
    launches0 = l1bench.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    kms = sess.profile(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = l1bench.launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    kms_long = sess.profile(prof_iters)
    kmode = sess.kernel_mode()
    tile = sess.tile_geometry() if kmode == 6 else None
    plan, plan_long = (sess.tile_plan(args.steps), sess.tile_plan(prof_iters)) if tile else ([], [])
    if tile and not (plan and plan_long):  # fewer than 6 timed iterations: two-iteration launches only
        tile = None
        kmode = 4
        kms = [kms[1], 0.0]  # (a tile session files those launches in the second slot)
        kms_long = [kms[0] * prof_iters / args.steps, 0.0]
    sess.end()
    out = {"ms_step": ms_total / args.steps, "ips": 1000.0 * args.steps / ms_total,
           "k1_ms": kms[0] / args.steps, "k2_ms": kms[1] / args.steps, "launches": int(launches),
           "k1_ms_long": kms_long[0] / prof_iters, "k2_ms_long": kms_long[1] / prof_iters,
           "kmode": kmode, "arith": arith}
    if tile:  # profile(): ms[0] = the tile launches, ms[1] = what is left after them
        out.update(tile=tile, tile_plan=plan, tile_plan_long=plan_long,
                   tile_ms=kms[0] / len(plan), tile_ms_long=kms_long[0] / len(plan_long), tile_launches=len(plan))
    return out


# FP64 flops per entry and iteration of the matrix-free FISTA step with S
# stages (fma = 2): the chains G^T x and G u, 3 per entry and stage each
# (the reference's rotation: 4 mul + 2 add per pair), plus r = sigma t - b
# (2), ||r||^2 (2), u = sigma ((1+beta) r - beta r') (4), y (3), y - g / L (2),
# the shrink (1) and ||x||_1 (1)
def flops_per_entry(stages):
    return 6 * stages + 15


def roofline_tile(t, info, stages, fp64_peak, fp64_src, hbm_peak, hbm_src):
    """The tile kernel (K iterations per launch) is bound by the FP64 pipe and
    its issue latency, not by HBM: the roofline is FP64 flops per launch over
    the measured fma throughput; the HBM side is reported beside it."""
    n = int(info.n)
    kmax, span, valid = t["tile"]
    plan = t["tile_plan"]
    k = sum(plan) / len(plan)  # iterations per launch of the timed region (20 = 10 + 10; 500 = 35 x 14 + 10)
    flops = flops_per_entry(stages) * n * k
    # x_k, x_{k-1}, sigma, b read once and two x written per launch (the tiles' overlapping
    # reads, (span - valid) / valid of the four inputs, hit L2: ncu DRAM bytes = 1.00 x 48n)
    byts = 48.0 * n
    ms, ms_long = t["tile_ms"], t["tile_ms_long"]
    achieved = flops / (ms * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("matrix_free:tile" + (":fma" if t.get("arith") == "fma" else ""))
        except Exception:
            traffic = None
    return {"bound": "fp64", "kernel": f"fista_tb ({kmax} FISTA iterations per launch on chip-resident tiles of "
                                       f"{span} entries, {valid} kept; matrix-free, residuals carried)",
            "launches": plan if len(plan) <= 8 else f"{plan.count(kmax)} x {kmax} + {[q for q in plan if q != kmax]}",
            "achieved": achieved, "peak": fp64_peak, "peak_source": fp64_src, "unit": "TFLOP/s",
            "frac": achieved / fp64_peak, "flops_per_launch": flops, "flops_per_entry_iteration": flops_per_entry(stages),
            "iterations_per_launch": k, "launch_ms": ms,
            "launch_ms_source": "CUDA events around every launch of the timed region",
            "launch_ms_long_run": ms_long, "achieved_long_run": flops / (ms_long * 1e-3) / 1e12,
            "traffic": traffic,
            "limiter": ("instruction issue at IPC 2.05 (issue slots 51.3 % busy, FP64 pipe 44.5 %): per iteration a "
                        "thread issues ~315 instructions for its 8 entries, 148 of them FP64; stalls: fixed-latency "
                        "dependencies, shuffle / shared-memory latency, the block barrier of the halo exchange "
                        "(profiles/r2_ncu_full_fista_tb3.txt, fma build); DRAM 6.44 GB per launch = 1.00 x 48n; the "
                        "pipe also carries the halo entries' work (own 240 of 256 per warp window, kept 1712 of 1920 per tile)"),
            "note": ("temporal blocking took the HBM bytes out of the iteration (48n bytes per 14 iterations instead "
                     "of per 2): this kernel is not HBM-bound, so its roofline is the FP64 one and roofline.hbm only "
                     "records how little of the memory system it needs; the HBM-bound two-iteration kernel (L1B_TB=0, "
                     "the sharded runs) reaches 0.93-1.00 of the measured copy bandwidth at 1870-2000 iter/s"),
            "hbm": {"achieved": byts / (ms * 1e-3) / 1e9, "peak": hbm_peak, "peak_source": hbm_src, "unit": "GB/s",
                    "frac": byts / (ms * 1e-3) / 1e9 / hbm_peak, "bytes_per_launch": byts},
            "hbm_gbs_ax_atr": byts / (ms * 1e-3) / 1e9}


def roofline(path, t, info, peak, peak_src):
    n, nnz = int(info.n), int(info.nnz)
    m_act = n  # banded: rows >= n are empty
    ptr_bytes = 4 if nnz < (1 << 32) else 8
    b1, b2, ipl = kernel_bytes(path, n, m_act, nnz, ptr_bytes, t.get("kmode"))
    if path == "matrix_free":
        names = (MF_KERNELS[t["kmode"]][2], "-")
        key1 = {4: "rc2", 3: "k1", 2: "stored"}[t["kmode"]]
    else:
        names = ("fista_k1 (A^T r_y + prox/momentum, CSC)", "fista_k2 (A x - b + residual momentum, CSR)")
        key1 = "k1"
    # per-launch time = per-iteration kernel time x iterations per launch
    dom = ((b1, t["k1_ms"] * ipl, names[0], key1) if t["k1_ms"] >= t["k2_ms"] else
           (b2, t["k2_ms"], names[1], "k2"))
    achieved = dom[0] / (dom[1] * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            key = f"{path}:{dom[3]}" + (":fma" if t.get("arith") == "fma" and path == "matrix_free" else "")
            traffic = json.load(open(tf)).get(key)
        except Exception:
            traffic = None
    long_ms = (t["k1_ms_long"] * ipl if dom[3] != "k2" else t["k2_ms_long"])
    if path == "matrix_free" and t.get("kmode") == 4:
        limiter = ("HBM streaming: ncu shows DRAM 6.44 GB per launch (1.00x algorithmic) at 80.5 % of its peak, the "
                   "FP64 pipe 45.7 % busy with the scaled rotations (profiles/r2_ncu_full_fista_rc2v_scaled.txt)" if t.get("arith") == "fma" else
                   "FP64 issue (separately rounded a*b+c): ncu shows the FP64 pipe at 76.5 % of peak and DRAM "
                   "at ~71 % (profiles/r1_ncu_full_fista_rc2v.txt)")
    else:
        limiter = "HBM streaming (profiles/r1_ncu_full_spmv_tma.txt)" if path == "sparse" else None
    return {"bound": "hbm", "kernel": dom[2], "achieved": achieved, "peak": peak, "limiter": limiter,
            "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
            "frac_of_8tbs": achieved / 8000.0, "bytes_per_launch": dom[0], "iterations_per_launch": ipl,
            "launch_ms": dom[1], "launch_ms_source": "CUDA events around every launch of the timed region",
            "launch_ms_long_run": long_ms, "achieved_long_run": dom[0] / (long_ms * 1e-3) / 1e9,
            "traffic": traffic,
            "hbm_gbs_ax_atr": (b1 + b2) / ((t["k1_ms"] * ipl + t["k2_ms"]) * 1e-3) / 1e9}


def run_reference(args, warmup, steps):
    """--impl reference / cpu_baseline: the reference's own fista_run
    (oracle/_ref/libl1ref.so, the unmodified /root/reference/proj/src sources
    compiled by oracle/Makefile; the plain-C oracle port where that build is
    absent) on the host cores, on the C4 configuration ITSELF: the instance is
    built by the reference's own generator at n = 2^27 (m = 2^28, ~20 GB of
    host memory) and `warmup` + `steps` FISTA iterations run in one fista_run;
    the timed region is the reference's own trace clock from the end of
    iteration `warmup` to the end of iteration `warmup + steps`.  Single
    threaded: the reference has no parallel code."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import REF_SO, Oracle, Reference

    kw = dict(C4)
    kw["n"] = args.n
    t_gen = time.perf_counter()
    if os.path.exists(REF_SO):
        lib, kind = Reference(), "reference"
        inst = lib.build_instance(**kw)
        t_gen = time.perf_counter() - t_gen
        tr, _ = inst.solve("fista", max_iters=warmup + steps)
        el = tr["elapsed_s"]
        it = list(tr["iter"])
        t = float(el[it.index(warmup + steps)] - el[it.index(warmup)])
    else:  # the oracle port (plain C restatement)
        lib, kind = Oracle(), "port"
        inst = lib.build_instance(**kw)
        t_gen = time.perf_counter() - t_gen
        t0 = time.perf_counter()
        lib.fista(inst, max_iters=warmup)
        t1 = time.perf_counter()
        lib.fista(inst, max_iters=warmup + steps)
        t = (time.perf_counter() - t1) - (t1 - t0)
    ips = steps / t
    return {
        "value": ips, "unit": UNIT, "cores": 1, "kind": kind,
        "sample": (f"{steps} FISTA iterations (after {warmup} untimed) of C4 itself "
                   f"(n=2^{int(math.log2(kw['n']))}, m=2n, 4 stages, q=1, s=n/1000, seed 3) through the "
                   f"reference's fista_run, single-threaded (the reference has no parallel code); "
                   f"instance built by the reference's generator in {t_gen:.1f} s (untimed)"),
        "seconds_timed": t, "generate_s": t_gen, "same_config": kw["n"] == C4["n"],
        "host_cores_total": os.cpu_count(),
    }


# the reference arm times at most this many C4 iterations (~8 s each on one
# host core): the whole --impl reference run then stays within a few minutes
REF_MAX_STEPS = 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # default K = the C4 config's own budget (500 FISTA iterations): the rate a
    # whole C4 run sustains under the power cap (a 20-iteration burst reads ~6 %
    # faster: the FP64-bound kernel runs at full clock until the cap engages)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--columns", dest="n", type=int, default=C4["n"],
                    help="global n, row-sharded across ranks when N > 1 (default C4: 2^27)")
    ap.add_argument("--arith", default="fma", choices=["fma", "exact"],
                    help="headline arithmetic of the matrix-free FISTA kernels")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sparse", action="store_true", help="skip the CSR/CSC leg (tuning runs)")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1-C3 side line")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the row-sharded NCCL driver even with one rank (plumbing check)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        steps = min(args.steps, REF_MAX_STEPS)
        cb = run_reference(args, warmup=min(args.warmup, 1), steps=steps)
        line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": steps, "steps_requested": args.steps, "warmup": args.warmup,
                "ms_per_step": 1000.0 / cb["value"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference generator, seed 3)", "impl": "reference",
                "config": {"workload": "C4 FISTA: n=2^27 cols x m=2^28 rows, 4 stages, q=1, s=n/1000, "
                                       "tau=1, seed 3 (the same instance as the GPU arm)"},
                "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch

    if world > 1 or args.force_dist:
        from paper_1503_03520_b200 import distributed

        return distributed.bench_main(args, world, rank, local)

    from paper_1503_03520_b200 import l1bench

    torch.cuda.set_device(local)
    kw = dict(C4)
    kw["n"] = args.n
    t0 = time.perf_counter()
    inst = l1bench.build_instance(device=local, lazy_sparse=True, **kw)
    gen_s = time.perf_counter() - t0
    peak, peak_src = peaks()
    fp64_peak = l1bench.fp64_peak(local)
    fp64_src = ("measured on this GPU by l1b_fp64_peak (independent fma chains, all SMs, best of 3); "
                "nominal 148 SMs x 64 lanes x 2 x 1.965 GHz = 37.2")

    def mf_roofline(t):
        if t["kmode"] == 6:
            return roofline_tile(t, info, kw["stages"], fp64_peak, fp64_src, peak, peak_src)
        return roofline("matrix_free", t, info, peak, peak_src)

    with ClockSampler(local) as clk:
        fused = time_path(inst, "matrix_free", args, arith=args.arith)
    info = inst.info  # builds nothing; CSR/CSC come with the first sparse use below
    rf = mf_roofline(fused)
    # the other arithmetic mode on the same instance (exact = the reference's bits)
    other = "exact" if args.arith == "fma" else "fma"
    with ClockSampler(local) as clk_other:
        alt = time_path(inst, "matrix_free", args, arith=other)
    alt_line = {"arith": other, "value": alt["ips"], "ms_per_step": alt["ms_step"],
                "roofline": mf_roofline(alt), "clocks": clk_other.summary()}
    # e2e before the CSR/CSC copy exists (37 GB of device memory at C4)
    e2e_line = e2e_more = None
    if not args.no_e2e:
        other = "exact" if args.arith == "fma" else "fma"
        e2e_line = e2e(inst, args.steps, local, arith=args.arith)
        e2e_more = {"serving_resident_operator": e2e(inst, args.steps, local, serving=True, arith=args.arith),
                    f"arith_{other}": e2e(inst, args.steps, local, arith=other)}
        if args.steps != C4_ITERS:  # the C4 run's own length beside the requested K
            e2e_more[f"k{C4_ITERS}"] = e2e(inst, C4_ITERS, local, arith=args.arith)
            e2e_more[f"k{C4_ITERS}_serving"] = e2e(inst, C4_ITERS, local, serving=True, arith=args.arith)
    if args.no_sparse:
        print(json.dumps({"metric": METRIC, "value": fused["ips"], "ms_per_step": fused["ms_step"],
                          "arith": args.arith, "roofline": rf, "clocks": clk.summary(),
                          "other_arith": alt_line, "note": "tuning run (--no-sparse)"}))
        return
    t0 = time.perf_counter()
    with ClockSampler(local) as clk_sparse:
        sparse = time_path(inst, "sparse", args, prof_iters=40)
    info = inst.materialize()  # refreshed: nnz of the CSR/CSC copy
    build_s = time.perf_counter() - t0
    rs = roofline("sparse", sparse, info, peak, peak_src)
    line = {
        "metric": METRIC, "value": fused["ips"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": fused["ms_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator on device, seed 3)",
        "config": {"workload": f"C4 FISTA: n=2^{int(math.log2(info.n))} cols x m=2^{int(math.log2(info.m))} rows, "
                               f"4 stages, nnz={info.nnz}, q=1, s=n/1000, tau=1, seed 3",
                   "l2": "inputs larger than L2 (no flush needed)", "parallelism": "single GPU",
                   "path": ("matrix-free (Givens stages in registers + warp shuffles, 256-bit loads); " +
                            (f"{sum(fused['tile_plan']) / len(fused['tile_plan']):g} FISTA iterations per launch "
                             f"(launches of up to {fused['tile'][0]}) on tiles held on chip (x halos "
                             f"exchanged between warps in shared memory, r_k carried between iterations): "
                             f"{48.0 * len(fused['tile_plan']) / sum(fused['tile_plan']):.2f}n bytes/iteration"
                             if fused["kmode"] == 6 else
                             "two FISTA iterations per launch, residuals recomputed, 24n bytes/iteration"
                             if fused["kmode"] == 4 else "one FISTA iteration per launch") +
                            ("; fused multiply-adds (arith='fma'; the tile kernel rotates in the scaled form, "
                             "prod cos carried by sigma): iterates within 1e-12 of the reference's "
                             "fista_run, same supports (tests/test_gpu_tile.py, tests/test_gpu_rc.py, "
                             "tests/test_gpu_configs.py)"
                             if args.arith == "fma" else
                             "; iterates bit-identical to the reference's fista_run")),
                   "arith": args.arith},
        "other_arith": alt_line,
        "gpu_launches": fused["launches"],
        "hbm_gbs_ax_atr": rf["hbm_gbs_ax_atr"],
        "kernels_ms_per_iteration": {"matrix_free": fused["k1_ms"]},
        "roofline": rf,
        "sparse_path": {"value": sparse["ips"], "ms_per_step": sparse["ms_step"],
                        "kernels_ms": {"fista_k1": sparse["k1_ms"], "fista_k2": sparse["k2_ms"]},
                        "hbm_gbs_ax_atr": rs["hbm_gbs_ax_atr"], "roofline": rs,
                        "gpu_launches": sparse["launches"], "csr_csc_build_s": build_s,
                        "note": "north-star CSR/CSC SpMV kernels (TMA bulk-copy pipeline)"},
        "generate_s": gen_s,
        "clocks": clk.summary(),
        "clocks_sparse": clk_sparse.summary(),
    }
    if e2e_line is not None:
        line["e2e"] = e2e_line
        line["e2e_more"] = e2e_more
    del inst
    if not args.no_configs:
        try:
            line["other_configs"] = small_configs()
        except Exception as e:  # reported, never silently substituted
            line["other_configs"] = {"error": str(e)}
    if not args.no_cpu:
        try:
            line["cpu_baseline"] = run_reference(args, warmup=1, steps=2)
        except Exception as e:  # reported, never silently substituted
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line))


def small_configs():
    """BASELINE.json's single-GPU side configurations C1-C3 (configs.py, same
    mapping): device time of the whole run / to the tolerance on this GPU.  The
    reference's CPU times beside them are in profiles/r1_configs.json."""
    import configs as C

    out = {}
    for name in ("c1", "c2", "c3"):
        r = C.run_gpu(name, C.CONFIGS[name])
        e = {"desc": r["desc"], "iterations": r["iterations"], "device_s": r["solve_device_s"],
             "status": r["status"], "rel_gap_final": r["rel_gap_final"]}
        if "time_to_target_s" in r:
            e["time_to_tolerance_s"] = r["time_to_target_s"]
        if "pcg_iterations" in r:
            e["pcg_iterations"] = r["pcg_iterations"]
        out[name] = e
    return out


def e2e(inst, steps, device, serving=False, arith="fma"):
    """Same metric through the public API from HOST buffers, every pass:
    upload sigma, b, x* (from_host -> l1b_problem_create), run K iterations
    (l1b_solve, default operator path) and copy x back -- all inside the timed
    region.  serving=True: the operator (sigma, stages) stays resident and a
    pass uploads only b (l1b_problem_set_rhs) before the solve.  arith: the
    l1b_solver_cfg.arith of the solve (the headline's; the other mode rides
    along in e2e_more)."""
    import torch

    from paper_1503_03520_b200 import l1bench

    def pinned(a):  # the caller's host data, in page-locked memory (set up untimed)
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = a
        return t.numpy()

    g = dict(sigma=pinned(inst.sigma()), b=pinned(inst.b), xs=inst.x_star)
    m, n, tau = inst.m, inst.n, inst.tau
    stages = [((4 - 1 - i) % 2, C4["theta"]) for i in range(4)]
    x = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    resident = None
    if serving:
        resident = l1bench.ProblemInstance.from_host(m, n, stages, g["sigma"], g["b"], tau, g["xs"].support,
                                                     g["xs"].values, device=device)
    times = []
    passes = 6 if steps <= 100 else 4  # short passes are noisier: median of five, else of three
    for rep in range(passes):  # pass 0 warms up (first-use pool growth / allocations); the rest are timed
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if serving:
            p = resident
            p.set_rhs(g["b"])
        else:
            p = l1bench.ProblemInstance.from_host(m, n, stages, g["sigma"], g["b"], tau, g["xs"].support,
                                                  g["xs"].values, device=device)
        tr = l1bench.fista_run(p, l1bench.SolverConfig(max_iters=steps, arith=arith), x)
        torch.cuda.synchronize()
        if rep:
            times.append(time.perf_counter() - t0)
        del p
    del resident
    t = sorted(times)[len(times) // 2]  # median
    h2d = 8 * m + (0 if serving else 8 * n + 12 * len(g["xs"].support))
    d2h = 8 * n + 48 * len(tr.samples)
    return {"value": steps / t, "unit": UNIT, "steps": steps, "arith": arith, "h2d_bytes_per_step": h2d / steps,
            "d2h_bytes_per_step": d2h / steps, "seconds": t, "seconds_passes": times,
            "includes": ("H2D of b from pinned host memory into the resident operator (l1b_problem_set_rhs), "
                         if serving else
                         "H2D of sigma/b/x* from pinned host buffers (l1b_problem_create), ") +
                        "K FISTA iterations (l1b_solve, matrix-free path), D2H of x and trace; wall clock, "
                        f"median of {passes - 1} identical passes after one warm-up pass"}


if __name__ == "__main__":
    main()
