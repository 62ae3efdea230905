#!/usr/bin/env python
"""bench.py -- condensed-KKT condense + factor + solve, ms per IPM iteration (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2] [--impl ours|reference]

One step = kkt_condense + kkt_factor + kkt_solve (LiftedKKT; refinement included) or
kkt_condense + kkt_factor + hykkt_solve (C3) on one synthetic instance per rank whose values
are re-drawn every step (successive IPM iterations on a fixed pattern).
Inputs are resident in HBM; L2 is flushed (256 MiB write) before every timed step and the
flush is outside the per-step CUDA-event window.  N > 1 (torchrun): every rank solves its own
instance (weak scaling, no data-path collective); value = max-over-ranks time / (N * K).
--workload C5: the 512-instance batch is partitioned over the ranks (strong scaling) and x is
gathered with NCCL at the end of every step; value = max-over-ranks time per batch iteration.

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
    ap.add_argument("--relax", default=None, help="amalgamation 'small,big,zero_frac' (perf tuning)")
    return ap.parse_args()


C5_TOTAL = 512


def workload(name, rank=0, redraw=0, world=1):
    """Instance(s) of rank `rank`.  C5: the rank's contiguous block of the 512-instance batch
    (instance k draws its values from seed 5000 + k (+1000 per redraw), so every partition
    reproduces the same instances).  Others: one instance per rank (weak scaling)."""
    from synth.generator import make_config, redraw_values, partition
    if name == "C5":
        a, b = partition(C5_TOTAL, world, rank)
        return make_config("C5", instance=a + 1000 * redraw, batch=b - a)
    inst = make_config(name, instance=rank)
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
    if inst.batch > 1:
        inst = inst.instance(0)
    import oracle  # noqa: F401
    _, _, sym = oracle_time(inst, 0.0)         # analysis once (untimed)
    for _ in range(args.warmup):
        pass
    t0 = time.perf_counter()
    ms_each = []
    nb = C5_TOTAL if args.workload == "C5" else 1
    for k in range(args.steps):
        it = workload(args.workload, 0, 1 + k % args.nvalues)
        if it.batch > 1:
            it = it.instance(k % it.batch)
        ms, cnt, _ = oracle_time(it, 0.0, sym)
        ms_each.append(ms * nb)        # C5: one batch iteration = 512 instance solves
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
                                      f"Cholesky + __float128-refined solve){' x 512 (one instance timed per step, scaled)' if nb > 1 else ''}, {total:.1f} s"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------ ours
def algorithmic_work(S, inst, refine_iters):
    """SURVEY §8(d) algorithmic work per instance."""
    n, m, nnzW, nnzJ = inst.n, inst.m, inst.nnzW, inst.nnzJ
    nnzK, nnzL = int(S.info["nnzK"]), int(S.info["nnzL"])
    condense_bytes = 8 * (nnzW + nnzJ + n + m) + 8 * nnzK
    trsv_bytes = 16 * nnzL + 24 * n
    resid_bytes = 24 * nnzW + 24 * nnzJ + 8 * (2 * n + m)
    pairs = 1 + refine_iters
    solve_bytes = pairs * trsv_bytes + (refine_iters + 1) * resid_bytes
    return dict(condense_bytes=condense_bytes, factor_flops=float(S.info["flops"]),
                trsv_bytes=trsv_bytes, resid_bytes=resid_bytes, solve_bytes=solve_bytes,
                trsv_pairs=pairs)


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
    batched = args.workload == "C5"
    inst = workload(args.workload, rank, 0, world)
    B = inst.batch
    hykkt = inst.m_eq > 0
    kw = {}
    if args.relax:
        a_, b_, c_ = args.relax.split(",")
        kw = dict(relax_small=int(a_), relax_big=int(b_), relax_zero_frac=float(c_))
    S = K.KKTSolver.from_instance(inst, **kw)
    S.bind(local)
    stream = torch.cuda.current_stream(dev)
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    # value sets cycled over steps (re-drawn values = successive IPM iterations, same pattern)
    sets = []
    for k in range(args.nvalues):
        it = workload(args.workload, rank, 1 + k, world)
        sets.append(dict(W=d(it.W_vals), J=d(it.J_vals), Sx=d(it.Sigma_x), Ss=d(it.Sigma_s),
                         b=d(it.b), r1=d(it.rbar1) if hykkt else None,
                         r2=d(it.rbar2) if hykkt else None, inst=it))
    x = torch.zeros((B, inst.n) if B > 1 else (inst.n,), dtype=torch.float64, device=dev)
    dy = torch.zeros(max(inst.m_eq, 1), dtype=torch.float64, device=dev)
    gathered = None
    if dist is not None and batched:
        from synth.generator import partition
        counts = [partition(C5_TOTAL, world, r)[1] - partition(C5_TOTAL, world, r)[0] for r in range(world)]
        assert len(set(counts)) == 1, "C5 multi-GPU run needs world | 512"
        gathered = torch.empty((C5_TOTAL, inst.n), dtype=torch.float64, device=dev)
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
        if gathered is not None:     # the only cross-GPU step: final gather of x (NCCL)
            dist.all_gather_into_tensor(gathered, x)
        if evs: evs[3].record(stream)
        return n1 + 2

    # kernels per step: condense + factor counted at enqueue; the solve graph's refinement loop
    # runs a data-dependent number of sweeps, so its count is read back after each warm-up step
    # (per value set) and reused for the timed steps, which stay free of host synchronisation
    per_set = {}

    for k in range(args.warmup):
        pre = step(sets[k % len(sets)])
        torch.cuda.synchronize()
        per_set[k % len(sets)] = pre + S.launch_count()
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
            step(sets[k % len(sets)], evs[k])
            launches += per_set.get(k % len(sets), max(per_set.values()))
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
    # batch: one step = one IPM iteration of the whole 512-instance batch (strong scaling);
    # otherwise every rank solves its own instance (weak scaling)
    value = total_ms / args.steps if batched else total_ms / (args.steps * world)
    # ---------------- e2e through host buffers (pinned) ----------------
    v0 = sets[0]["inst"]
    pin = lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory()
    e2e_ms = None
    h2d = d2h = 0
    if not hykkt:
        hW, hJ, hSx, hSs, hb = (pin(v0.W_vals), pin(v0.J_vals), pin(v0.Sigma_x), pin(v0.Sigma_s), pin(v0.b))
        hx = torch.zeros(tuple(x.shape), dtype=torch.float64).pin_memory()
        call = lambda: K.kkt_step_host(S.h, hW, hJ, hSx, hSs, None, inst.delta_w, inst.delta_c,
                                       inst.gamma, hb, hx, args.max_refine, 0.0)
        for _ in range(2):
            call()
        e0, e1 = ev(), ev()
        ts = []
        for k in range(args.steps):
            flush.fill_(float(k))
            e0.record(stream)
            call()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        e2e_tot = float(np.sum(ts))
        if dist:
            t = torch.tensor([e2e_tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_tot = float(t.item())
        e2e_ms = e2e_tot / args.steps if batched else e2e_tot / (args.steps * world)
        h2d = 8 * B * (inst.nnzW + inst.nnzJ + inst.n + (inst.m - inst.m_eq) + inst.n)
        d2h = 8 * B * inst.n
    # ---------------- roofline ----------------
    ph_mean = ph.mean(0)
    work = algorithmic_work(S, inst, max(info["refine_iters"], 0))
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    pk = json.load(open(pk_path)) if os.path.exists(pk_path) else {}
    fp64 = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")))
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    hbm_note = "MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in pk else "fallback 6650 GB/s"
    f_ach = B * work["factor_flops"] / (ph_mean[1] * 1e-3) / 1e12
    roof_factor = {"bound": "tensor", "achieved": f_ach, "peak": fp64["dmma_tflops"], "unit": "TFLOP/s",
                   "frac": f_ach / fp64["dmma_tflops"], "traffic": None,
                   "kernel": "kkt_factor (factor_small_kernel + factor_big_kernel)",
                   "work": "B x sum_j c_j^2 flops per call",
                   "peak_note": "FP64 DMMA (mma.sync m8n8k4) measured by tools/fp64_peaks.cu, profiles/r01_fp64_peaks.json"}
    s_ach = B * work["solve_bytes"] / (ph_mean[2] * 1e-3) / 1e9
    roof_solve = {"bound": "hbm", "achieved": s_ach, "peak": hbm_peak, "unit": "GB/s",
                  "frac": s_ach / hbm_peak, "traffic": None,
                  "kernel": ("hykkt_solve" if hykkt else "kkt_solve") + " (fwd/bwd trsv kernels + dd residual)",
                  "work": f"B x [{work['trsv_pairs']} trsv pairs x 16 nnz(L) + residual passes] bytes",
                  "peak_note": hbm_note}
    c_ach = B * work["condense_bytes"] / (ph_mean[0] * 1e-3) / 1e9
    roof_cond = {"bound": "hbm", "achieved": c_ach, "peak": hbm_peak, "unit": "GB/s", "frac": c_ach / hbm_peak,
                 "traffic": None, "kernel": "condense_kernel (+dweights_kernel)"}
    roofs = {"condense": roof_cond, "factor": roof_factor, "solve": roof_solve}
    tpath = os.path.join(ROOT, "profiles", f"r01_traffic_{args.workload}.json")
    if os.path.exists(tpath):  # DRAM bytes per phase from one ncu capture (cold caches per launch)
        tr = json.load(open(tpath))
        for k_, r_ in roofs.items():
            r_["traffic"] = tr["dram_bytes_per_step"].get(k_) / max(B, 1) if tr["dram_bytes_per_step"].get(k_) else None
            r_["traffic_note"] = "ncu dram__bytes_read+write per step of this phase (" + tr["source"] + ")"
    dom = ["condense", "factor", "solve"][int(np.argmax(ph_mean))]
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": False, "scaling": "strong" if batched else "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, synth/)",
           "config": {"workload": f"{args.workload}: {describe(args.workload)}", "n": inst.n,
                      "m": inst.m, "m_eq": inst.m_eq, "batch_per_gpu": B,
                      "nnzK": int(S.info["nnzK"]), "nnzL": int(S.info["nnzL"]),
                      "flops": S.info["flops"], "nsuper": S.info["nsuper"],
                      "tree_height": S.info["tree_height"],
                      "l2": "flushed (256 MiB write) before every step, outside the event window",
                      "max_refine": args.max_refine,
                      "parallelism": f"{'batch partition' if batched else 'instance per GPU'} x{world}"},
           "phases_ms": {n_: float(v_) for n_, v_ in zip(["condense", "factor", "solve"], ph_mean)},
           "refine_iters": info["refine_iters"], "cg_iters": info["cg_iters"],
           "bwd_err": info["bwd_err"], "analyze_ms": S.info["analyze_ms"],
           "wall_s_timed": t_wall,
           "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
           "gpu_launches": launches,
           "roofline": dict(roofs[dom], phase=dom),
           "roofline_phases": roofs,
           "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        one = inst.instance(0) if B > 1 else inst
        ms, cnt, _ = oracle_time(one, args.cpu_sample_s)
        out["cpu_baseline"] = {"value": ms * B, "unit": UNIT, "cores": 1, "kind": "oracle",
                               "sample": f"{cnt} oracle IPM iterations of one {args.workload} instance "
                                         f"(condense + Cholesky + __float128 refined solve), "
                                         f"~{args.cpu_sample_s:.0f} s budget" + (f"; x{B} for the batch" if B > 1 else "")}
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
