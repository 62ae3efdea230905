#!/usr/bin/env python
"""bench.py -- condensed-KKT condense + factor + solve, ms per IPM iteration (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2] [--impl ours|reference]

One step = kkt_condense + kkt_factor + kkt_solve (LiftedKKT; refinement included) or
kkt_condense + kkt_factor + hykkt_solve (C3) on one synthetic instance per rank whose values
are re-drawn every step (successive IPM iterations on a fixed pattern).
Inputs are resident in HBM; L2 is flushed (256 MiB write) before every timed step and the
flush is outside the per-step CUDA-event window.  N > 1 (torchrun): every rank solves its own
instance (weak scaling, no data-path collective); value = max-over-ranks time / (N * K).

--impl reference times the CPU oracle (oracle/, plain C, __float128) on the same workload --
there is no installable reference implementation for this paper.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

METRIC = "condensed KKT condense+factor+solve ms/IPM-iter"
UNIT = "ms"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--max-refine", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=15.0)
    ap.add_argument("--nvalues", type=int, default=4, help="distinct value sets cycled over steps")
    return ap.parse_args()


def workload(name, rank=0, redraw=0):
    from synth.generator import make_config, redraw_values
    inst = make_config(name, instance=0)
    if redraw:
        inst = redraw_values(inst, 100000 * (rank + 1) + redraw)
    return inst


def describe(name):
    from synth.generator import CONFIGS
    return CONFIGS.get(name, name)


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 4 + k and s[4 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------ oracle
def oracle_step(inst):
    """One IPM iteration of the CPU oracle: condense -> Cholesky -> refined solve (ordering and
    symbolic analysis are once-per-pattern and excluded, as for the GPU path)."""
    import oracle
    K = oracle.condense(inst)
    return K


def oracle_time(inst, budget_s, symbolic=None):
    import oracle
    t0 = time.perf_counter()
    if symbolic is None:
        K = oracle.condense(inst)
        perm = oracle.md_order(inst.n, K[0], K[1])
        _, _, Lp, Li = oracle.symbolic(inst.n, K[0], K[1], perm, want_pattern=True)
        symbolic = (perm, Lp, Li)
    perm, Lp, Li = symbolic
    times = []
    t_start = time.perf_counter()
    while True:
        t = time.perf_counter()
        K = oracle.condense(inst)
        Lx, fail = oracle.cholesky(inst.n, K[0], K[1], K[2], perm, Lp, Li)
        if inst.m_eq:
            oracle.hykkt(inst, Lp, Li, Lx, perm, inst.rbar1, inst.rbar2, 1e-12, 2000, 2)
        else:
            oracle.solve_refined(inst, Lp, Li, Lx, perm, inst.b, max_sweeps=10, stop_rel=2.2e-16)
        times.append(time.perf_counter() - t)
        if time.perf_counter() - t_start >= budget_s or len(times) >= 1000:
            break
    return float(np.mean(times)) * 1e3, len(times), symbolic


def run_reference(args, rank, world):
    if rank != 0:
        return
    inst = workload(args.workload)
    import oracle  # noqa: F401
    _, _, sym = oracle_time(inst, 0.0)         # analysis once (untimed)
    for _ in range(args.warmup):
        pass
    t0 = time.perf_counter()
    ms_each = []
    for k in range(args.steps):
        ms, cnt, _ = oracle_time(workload(args.workload, 0, 1 + k % args.nvalues), 0.0, sym)
        ms_each.append(ms)
    total = time.perf_counter() - t0
    v = float(np.mean(ms_each))
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.workload}: {describe(args.workload)}", "n": inst.n,
                      "m": inst.m, "m_eq": inst.m_eq},
           "impl": "reference",
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{args.steps} full oracle IPM iterations (condense + "
                                      f"Cholesky + __float128-refined solve), {total:.1f} s"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------ ours
def run_ours(args, rank, world):
    import torch
    import paper_2405_14236_b200 as K

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    inst = workload(args.workload, rank)
    hykkt = inst.m_eq > 0
    S = K.KKTSolver.from_instance(inst)
    S.bind(local)
    stream = torch.cuda.current_stream(dev)
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    # value sets cycled over steps (re-drawn values = successive IPM iterations)
    sets = []
    for k in range(args.nvalues):
        it = workload(args.workload, rank, 1 + k)
        sets.append(dict(W=d(it.W_vals), J=d(it.J_vals), Sx=d(it.Sigma_x), Ss=d(it.Sigma_s),
                         b=d(it.b), r1=d(it.rbar1) if hykkt else None,
                         r2=d(it.rbar2) if hykkt else None, inst=it))
    x = torch.zeros(inst.n, dtype=torch.float64, device=dev)
    dy = torch.zeros(max(inst.m_eq, 1), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step(v, evs=None):
        if evs: evs[0].record(stream)
        S.condense(v["W"], v["J"], v["Sx"], v["Ss"], None, inst.delta_w, inst.delta_c, inst.gamma)
        n1 = S.launch_count()
        if evs: evs[1].record(stream)
        S.factor()
        if evs: evs[2].record(stream)
        if hykkt:
            S.hykkt_solve(v["r1"], v["r2"], x, dy, 1e-12, 0, 2)
        else:
            S.solve(v["b"], x, args.max_refine, 0.0)
        n3 = S.launch_count()
        if evs: evs[3].record(stream)
        return n1 + 1 + n3

    for k in range(args.warmup):
        step(sets[k % len(sets)])
    torch.cuda.synchronize()
    info = S.sync_info()
    if info["status"] != 0:
        raise RuntimeError(f"warm-up solve failed: {info}")
    # ---------------- timed region ----------------
    evs = [[ev() for _ in range(4)] for _ in range(args.steps)]
    launches = 0
    if dist: dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.fill_(float(k))                  # L2 flush, outside the event window
            launches += step(sets[k % len(sets)], evs[k])
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if dist: dist.barrier()
    torch.cuda.synchronize()
    ph = np.array([[evs[k][0].elapsed_time(evs[k][1]), evs[k][1].elapsed_time(evs[k][2]),
                    evs[k][2].elapsed_time(evs[k][3])] for k in range(args.steps)])
    total_ms = float(ph.sum())
    info = S.sync_info()
    if dist:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_solve = total_ms / (args.steps * world)
    # ---------------- e2e through host buffers (pinned) ----------------
    v0 = sets[0]["inst"]
    pin = lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory()
    hW, hJ, hSx, hSs, hb = (pin(v0.W_vals), pin(v0.J_vals), pin(v0.Sigma_x), pin(v0.Sigma_s), pin(v0.b))
    hx = torch.zeros(inst.n, dtype=torch.float64).pin_memory()
    e2e_ms = None
    if not hykkt:
        for _ in range(2):
            K.kkt_step_host(S.h, hW, hJ, hSx, hSs, None, inst.delta_w, inst.delta_c, inst.gamma, hb, hx,
                            args.max_refine, 0.0)
        e0, e1 = ev(), ev()
        ts = []
        for k in range(args.steps):
            flush.fill_(float(k))
            e0.record(stream)
            K.kkt_step_host(S.h, hW, hJ, hSx, hSs, None, inst.delta_w, inst.delta_c, inst.gamma, hb, hx,
                            args.max_refine, 0.0)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        e2e_tot = float(np.sum(ts))
        if dist:
            t = torch.tensor([e2e_tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_tot = float(t.item())
        e2e_ms = e2e_tot / (args.steps * world)
    h2d = 8 * (inst.nnzW + inst.nnzJ + inst.n + (inst.m - inst.m_eq) + inst.n)
    d2h = 8 * inst.n
    # ---------------- roofline of the dominant phase ----------------
    ph_mean = ph.mean(0)
    names = ["condense", "factor", "solve"]
    dom = int(np.argmax(ph_mean))
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    fp64 = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")))
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    nnzK = int(S.info["nnzK"])
    if names[dom] == "factor":
        achieved = S.info["flops"] / (ph_mean[1] * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": fp64["dfma_tflops"], "unit": "TFLOP/s",
                "frac": achieved / fp64["dfma_tflops"], "traffic": None, "kernel": "factor_kernel",
                "note": "FP64 DFMA peak measured by tools/fp64_peaks.cu (profiles/r01_fp64_peaks.json)"}
    elif names[dom] == "condense":
        byts = 8 * (inst.nnzW + inst.nnzJ + inst.n + inst.m) + 8 * nnzK
        achieved = byts / (ph_mean[0] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": None, "kernel": "condense_kernel"}
    else:
        sweeps = 1 + 2 * max(info["refine_iters"], 0) if not hykkt else None
        byts = 16 * S.info["nnzL"] + 24 * inst.n
        achieved = byts / (ph_mean[2] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": None, "kernel": "solve (fwd+bwd+refine)",
                "note": "algorithmic bytes of ONE trsv pair over the whole solve phase"}
    out = {"metric": METRIC, "value": ms_per_solve, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": f"{args.workload}: {describe(args.workload)}", "n": inst.n,
                      "m": inst.m, "m_eq": inst.m_eq, "nnzK": nnzK, "nnzL": int(S.info["nnzL"]),
                      "flops": S.info["flops"], "nsuper": S.info["nsuper"],
                      "l2": "flushed (256 MiB write) before every step, outside the event window",
                      "max_refine": args.max_refine, "parallelism": f"instances x{world}"},
           "phases_ms": {n_: float(v) for n_, v in zip(names, ph_mean)},
           "refine_iters": info["refine_iters"], "cg_iters": info["cg_iters"],
           "bwd_err": info["bwd_err"], "analyze_ms": S.info["analyze_ms"],
           "wall_s_timed": t_wall,
           "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": h2d if e2e_ms else 0,
                   "d2h_bytes_per_step": d2h if e2e_ms else 0},
           "gpu_launches": launches,
           "roofline": roof,
           "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ms, cnt, _ = oracle_time(inst, args.cpu_sample_s)
        out["cpu_baseline"] = {"value": ms, "unit": UNIT, "cores": 1, "kind": "oracle",
                               "sample": f"{cnt} oracle IPM iterations of {args.workload} "
                                         f"(condense + Cholesky + __float128 refined solve), "
                                         f"~{args.cpu_sample_s:.0f} s budget"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    S.close()
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if world != args.gpus and "WORLD_SIZE" not in os.environ:
        world = 1
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
