#!/usr/bin/env python
"""bench.py -- condensed-KKT condense + factor + solve, ms per IPM iteration (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl ours|reference]

One step = kkt_condense + kkt_factor + kkt_solve (LiftedKKT; refinement included) or
kkt_condense + kkt_factor + hykkt_solve (C3) on synthetic values re-drawn every step
(successive IPM iterations on a fixed pattern).  Inputs are resident in HBM; L2 is
flushed (256 MiB write) before every timed step, outside the per-step CUDA-event window.

Default workload: C4 (78,484-bus ACOPF, LiftedKKT), the largest single-GPU configuration of
BASELINE.json (configs[3]).  Multi-GPU (one process per GPU; `--gpus N` without torchrun
re-launches itself under torch.distributed.run):
  * C1..C4, C6: replicas only (one KKT system stays on one GPU) -- every rank
    solves its own instance; value = per-iteration time, max over ranks ("scaling": "weak");
  * C5: the 512-instance batch is partitioned contiguously over the ranks and x is gathered to
    rank 0 (NCCL gather) at the end of every step; value = time per batch iteration, max over
    ranks ("scaling": "strong").

--impl reference times the CPU oracle (oracle/, plain C, __float128 accumulation) on the same
workload, config dict, metric and unit -- there is no installable reference implementation for
this paper.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

METRIC = "condensed KKT condense+factor+solve ms/IPM-iter"
UNIT = "ms"
C5_TOTAL = 512
L2_NOTE = "flushed (256 MiB write) before every step, outside the event window"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--max-refine", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0,
                    help="budget of timed oracle iterations for cpu_baseline (after its analysis)")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: wall budget of the timed oracle steps")
    ap.add_argument("--nvalues", type=int, default=4, help="distinct value sets cycled over steps")
    ap.add_argument("--relax", default=None, help="amalgamation 'small,big,zero_frac' (perf tuning)")
    return ap.parse_args()


def workload(name, rank=0, redraw=0, world=1):
    """Instance(s) of rank `rank`.  C5: the rank's contiguous block of the 512-instance batch
    (instance k draws its values from seed 5000 + k (+1000 per redraw), so every partition
    reproduces the same instances).  Others: one instance per rank (replicas)."""
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


def config_of(args, inst, world):
    """The config dict both arms print (identical keys and values for the same command)."""
    batched = args.workload == "C5"
    return {"workload": f"{args.workload}: {describe(args.workload)}", "n": int(inst.n),
            "m": int(inst.m), "m_eq": int(inst.m_eq),
            "batch_total": C5_TOTAL if batched else world,
            "l2": L2_NOTE, "max_refine": args.max_refine,
            "parallelism": (f"batch partition x{world}" if batched else f"replicas x{world}")}


def cpu_info():
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "host": socket.gethostname()}


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
            self._stop.wait(0.1)

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
def oracle_analysis(inst):
    """Once-per-pattern oracle analysis: ordering + symbolic (timed separately, not per iteration)."""
    import oracle
    t0 = time.perf_counter()
    K = oracle.condense(inst)                      # pattern of K (values unused here)
    t1 = time.perf_counter()
    perm = oracle.md_order(inst.n, K[0], K[1])
    t2 = time.perf_counter()
    _, _, Lp, Li = oracle.symbolic(inst.n, K[0], K[1], perm, want_pattern=True)
    t3 = time.perf_counter()
    return (perm, Lp, Li), {"pattern_ms": (t1 - t0) * 1e3, "ordering_ms": (t2 - t1) * 1e3,
                            "symbolic_ms": (t3 - t2) * 1e3}


def oracle_iteration(inst, sym):
    """One oracle IPM iteration: condense -> Cholesky -> refined solve (or HyKKT), per phase (ms)."""
    import oracle
    perm, Lp, Li = sym
    t0 = time.perf_counter()
    K = oracle.condense(inst)
    t1 = time.perf_counter()
    Lx, fail = oracle.cholesky(inst.n, K[0], K[1], K[2], perm, Lp, Li)
    t2 = time.perf_counter()
    if inst.m_eq:
        oracle.hykkt(inst, Lp, Li, Lx, perm, inst.rbar1, inst.rbar2, 1e-12, 2000, 2)
    else:
        oracle.solve_refined(inst, Lp, Li, Lx, perm, inst.b, max_sweeps=10, stop_rel=2.2e-16)
    t3 = time.perf_counter()
    return {"condense": (t1 - t0) * 1e3, "factor": (t2 - t1) * 1e3, "solve": (t3 - t2) * 1e3,
            "total": (t3 - t0) * 1e3}


def oracle_baseline(args, inst, budget_s, threads=1):
    """cpu_baseline: the oracle as it stands on the host cores, bounded sample.  One instance per
    thread when threads > 1 (C5: embarrassingly parallel batch)."""
    one = inst.instance(0) if inst.batch > 1 else inst
    sym, ana = oracle_analysis(one)
    per = []
    t_start = time.perf_counter()
    while True:
        per.append(oracle_iteration(one, sym))
        if time.perf_counter() - t_start >= budget_s or len(per) >= 200:
            break
    ph = {k: float(np.mean([p[k] for p in per])) for k in per[0]}
    out = {"iters": len(per), "phases_ms": ph, "analysis_ms": ana, "iter_ms": ph["total"]}
    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor
        insts = [inst.instance(k % inst.batch) for k in range(2 * threads)]
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:   # ctypes releases the GIL inside the C oracle
            list(ex.map(lambda it: oracle_iteration(it, sym), insts))
        dt = time.perf_counter() - t0
        out["parallel"] = {"threads": threads, "instances": len(insts), "wall_s": dt,
                           "ms_per_instance": dt * 1e3 / len(insts)}
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return   # rank 0 alone runs the (CPU) reference arm; other ranks exit 0
    inst0 = workload(args.workload, 0, 0, 1)
    one = inst0.instance(0) if inst0.batch > 1 else inst0
    nb = C5_TOTAL if args.workload == "C5" else 1
    sym, ana = oracle_analysis(one)                   # once per pattern, untimed
    warm = min(args.warmup, 1)                        # the oracle has no caches to warm
    for k in range(warm):
        oracle_iteration(one, sym)
    sets = []
    for k in range(min(args.nvalues, args.steps)):   # same re-drawn value sets as our arm
        it = workload(args.workload, 0, 1 + k, 1)
        sets.append(it.instance(k % it.batch) if it.batch > 1 else it)
    per = []
    t0 = time.perf_counter()
    for k in range(args.steps):
        per.append(oracle_iteration(sets[k % len(sets)], sym))
        if time.perf_counter() - t0 >= args.ref_budget_s:
            break
    total = time.perf_counter() - t0
    v = float(np.mean([p["total"] for p in per])) * nb   # C5: one batch iteration = 512 solves
    phases = {k: float(np.mean([p[k] for p in per])) * nb for k in ("condense", "factor", "solve")}
    sample = (f"{len(per)} of {args.steps} requested oracle IPM iterations (condense + Cholesky + "
              f"__float128-refined solve) in {total:.1f} s (budget {args.ref_budget_s:.0f} s), "
              f"{warm} warm-up" + ("; one instance per step, x512 for the batch" if nb > 1 else ""))
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": len(per),
           "warmup": warm, "ms_per_step": v, "higher_is_better": False,
           "scaling": "strong" if nb > 1 else "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded generator, synth/)",
           "config": config_of(args, inst0, world), "impl": "reference",
           "phases_ms": phases, "oracle_analysis_ms": ana,
           "cpu_baseline": dict({"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                                 "sample": sample}, **cpu_info()),
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------ ours
def algorithmic_work(info, inst, refine_iters, cg_iters=0):
    """SURVEY §8(d) algorithmic work per instance.  HyKKT (m_eq > 0): every pass
    runs 2 trsv pairs (z = K_gamma^-1 s, the final dx) plus one per Krylov iteration; cg_iters is
    the Krylov total over all passes (kkt_hykkt_stats); the G / G^T products are not counted (a
    lower bound); refine_iters = outer passes after the first, each preceded by one dd residual."""
    n, m, nnzW, nnzJ = inst.n, inst.m, inst.nnzW, inst.nnzJ
    nnzK, nnzL = int(info["nnzK"]), int(info["nnzL"])
    condense_bytes = 8 * (nnzW + nnzJ + n + m) + 8 * nnzK
    trsv_bytes = 16 * nnzL + 24 * n
    resid_bytes = 24 * nnzW + 24 * nnzJ + 8 * (2 * n + m)
    if inst.m_eq > 0:
        pairs = 2 * (1 + refine_iters) + cg_iters
        resid_passes = refine_iters
    else:
        pairs = 1 + refine_iters
        resid_passes = refine_iters + 1
    solve_bytes = pairs * trsv_bytes + resid_passes * resid_bytes
    return dict(condense_bytes=condense_bytes, factor_flops=float(info["flops"]),
                factor_flops_large=float(info["flops_huge"]),
                trsv_bytes=trsv_bytes, resid_bytes=resid_bytes, solve_bytes=solve_bytes,
                trsv_pairs=pairs, resid_passes=resid_passes)


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
    gather_list = None
    if dist is not None and batched:
        from synth.generator import partition
        counts = [partition(C5_TOTAL, world, r)[1] - partition(C5_TOTAL, world, r)[0] for r in range(world)]
        assert len(set(counts)) == 1, "C5 multi-GPU run needs world | 512"
        if rank == 0:   # x of every rank lands here: the only cross-GPU step (final gather)
            gather_list = [torch.empty_like(x) for _ in range(world)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step(v, evs=None):
        if evs: evs[0].record(stream)
        S.condense(v["W"], v["J"], v["Sx"], v["Ss"], None, inst.delta_w, inst.delta_c, inst.gamma)
        if evs: evs[1].record(stream)
        S.factor()
        n1 = S.launch_count()       # condense + factor kernels (the counter restarts at condense)
        if evs: evs[2].record(stream)
        if hykkt:
            S.hykkt_solve(v["r1"], v["r2"], x, dy, 1e-12, 0, 2)
        else:
            S.solve(v["b"], x, args.max_refine, 0.0)
        if dist is not None and batched:
            dist.gather(x, gather_list, dst=0)
        if evs: evs[3].record(stream)
        return n1

    # kernels per step: condense + factor counted at enqueue; the solve's data-dependent part is
    # read back after each warm-up step (per value set) and reused for the timed steps, which
    # stay free of host synchronisation
    per_set = {}
    for k in range(max(args.warmup, len(sets))):
        pre = step(sets[k % len(sets)])
        torch.cuda.synchronize()
        per_set[k % len(sets)] = pre + S.launch_count()
    torch.cuda.synchronize()
    info = S.sync_info()
    if info["status"] != 0:
        raise RuntimeError(f"warm-up solve failed: {info}")
    # ---------------- timed region ----------------
    evs = [[ev() for _ in range(4)] for _ in range(args.steps)]
    fph = []
    launches = 0
    if dist: dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.fill_(float(k))                  # L2 flush, outside the event window
            step(sets[k % len(sets)], evs[k])
            launches += per_set[k % len(sets)]
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if dist: dist.barrier()
    torch.cuda.synchronize()
    ph = np.array([[evs[k][0].elapsed_time(evs[k][1]), evs[k][1].elapsed_time(evs[k][2]),
                    evs[k][2].elapsed_time(evs[k][3])] for k in range(args.steps)])
    total_ms = float(ph.sum())
    info = S.sync_info()
    # factor split by supernode class (events inside kkt_factor), measured on the last step and
    # on separate timed factor calls with the same flush discipline
    for k in range(min(args.steps, 10)):
        flush.fill_(float(k))
        S.condense(sets[k % len(sets)]["W"], sets[k % len(sets)]["J"], sets[k % len(sets)]["Sx"],
                   sets[k % len(sets)]["Ss"], None, inst.delta_w, inst.delta_c, inst.gamma)
        S.factor()
        fph.append(S.factor_phase_ms())
    fph = np.array(fph)
    if dist:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = total_ms / args.steps     # ms per IPM iteration (C5: per batch iteration)
    # ---------------- e2e through host buffers (pinned) ----------------
    v0 = sets[0]["inst"]
    pin = lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory()
    e2e_ms = None
    h2d = d2h = 0
    if True:
        hW, hJ, hSx, hSs = (pin(v0.W_vals), pin(v0.J_vals), pin(v0.Sigma_x), pin(v0.Sigma_s))
        hx = torch.zeros(tuple(x.shape), dtype=torch.float64).pin_memory()
        if not hykkt:
            hb = pin(v0.b)
            call = lambda: K.kkt_step_host(S.h, hW, hJ, hSx, hSs, None, inst.delta_w, inst.delta_c,
                                           inst.gamma, hb, hx, args.max_refine, 0.0)
        else:
            # HyKKT has no host-buffer entry point: the public calls on device buffers, with the
            # pinned-host copies of the step's inputs and of (dx, dy) on the handle's stream
            hr1, hr2 = pin(v0.rbar1), pin(v0.rbar2)
            hdy = torch.zeros(tuple(dy.shape), dtype=torch.float64).pin_memory()
            dev_in = [torch.empty_like(t_, device=dev) for t_ in (hW, hJ, hSx, hSs, hr1, hr2)]

            def call():
                for dd_, hh_ in zip(dev_in, (hW, hJ, hSx, hSs, hr1, hr2)):
                    dd_.copy_(hh_, non_blocking=True)
                S.condense(dev_in[0], dev_in[1], dev_in[2], dev_in[3], None, inst.delta_w, inst.delta_c,
                           inst.gamma)
                S.factor()
                S.hykkt_solve(dev_in[4], dev_in[5], x, dy, 1e-12, 0, 2)
                hx.copy_(x, non_blocking=True)
                hdy.copy_(dy, non_blocking=True)
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
        e2e_ms = e2e_tot / args.steps
        if not hykkt:
            h2d = 8 * B * (inst.nnzW + inst.nnzJ + inst.n + (inst.m - inst.m_eq) + inst.n)
            d2h = 8 * B * inst.n
        else:
            h2d = sum(8 * t_.numel() for t_ in (hW, hJ, hSx, hSs, hr1, hr2))
            d2h = 8 * (hx.numel() + hdy.numel())
    # ---------------- roofline ----------------
    ph_mean = ph.mean(0)
    krylov_total = S.hykkt_stats()["krylov_total"] if hykkt else 0
    work = algorithmic_work(S.info, inst, max(info["refine_iters"], 0), krylov_total)
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    pk = json.load(open(pk_path)) if os.path.exists(pk_path) else {}
    fp64 = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")))
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    hbm_note = ("MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in pk else
                "fallback 6650 GB/s (B200_PROFILING.md)")
    dmma_note = "FP64 DMMA (mma.sync m8n8k4 -> DMMA.8x8x4) measured by tools/fp64_peaks.cu, profiles/r01_fp64_peaks.json"
    f_ach = B * work["factor_flops"] / (ph_mean[1] * 1e-3) / 1e12
    roofs = {}
    roofs["condense"] = {"bound": "hbm", "achieved": B * work["condense_bytes"] / (ph_mean[0] * 1e-3) / 1e9,
                         "peak": hbm_peak, "unit": "GB/s", "traffic": None,
                         "kernel": "condense_kernel (+dweights_kernel)",
                         "work": "B x [8 (nnzW+nnzJ+n+m) + 8 nnzK] bytes", "peak_note": hbm_note}
    roofs["factor"] = {"bound": "tensor", "achieved": f_ach, "peak": fp64["dmma_tflops"], "unit": "TFLOP/s",
                       "traffic": None, "kernel": "kkt_factor (all supernode classes)",
                       "work": "B x sum_j c_j^2 flops", "peak_note": dmma_note}
    fl_ms = fph.mean(0) if len(fph) else np.zeros(2)
    if work["factor_flops_large"] > 0 and fl_ms[1] > 0:
        ach = B * work["factor_flops_large"] / (fl_ms[1] * 1e-3) / 1e12
        roofs["factor_large"] = {
            "bound": "tensor", "achieved": ach, "peak": fp64["dmma_tflops"], "unit": "TFLOP/s",
            "traffic": None, "kernel": "tile_factor_kernel (large supernodes: 64x64 tile DAG, DMMA)",
            "work": f"B x {work['factor_flops_large']:.4g} flops (sum over large supernodes of "
                    "sum_t (r - t)^2)",
            "threshold": "front > 25600 doubles (beyond one CTA's shared memory) and ancestors; "
                         f"{S.info['nsuper_huge']} supernodes",
            "flop_share": work["factor_flops_large"] / max(work["factor_flops"], 1.0),
            "time_ms": float(fl_ms[1]), "time_share": float(fl_ms[1] / max(fl_ms.sum(), 1e-9)),
            "peak_note": dmma_note}
    roofs["solve"] = {"bound": "hbm", "achieved": B * work["solve_bytes"] / (ph_mean[2] * 1e-3) / 1e9,
                      "peak": hbm_peak, "unit": "GB/s", "traffic": None,
                      "kernel": ("hykkt_solve" if hykkt else "kkt_solve") + " (fwd/bwd trsv kernels + dd residual)",
                      "work": f"B x [{work['trsv_pairs']} trsv pairs x (16 nnz(L) + 24 n) + "
                              f"{work['resid_passes']} dd residual passes] bytes"
                              + (f" (HyKKT: {krylov_total} Krylov iterations over all passes + 2 pairs per pass; G, G^T products not counted)"
                                 if hykkt else ""),
                      "peak_note": hbm_note}
    for r_ in roofs.values():
        r_["frac"] = r_["achieved"] / r_["peak"]
    tpath = os.path.join(ROOT, "profiles", f"r02_traffic_{args.workload}.json")
    if os.path.exists(tpath):  # DRAM bytes per phase / kernel from one ncu capture (cold caches)
        tr = json.load(open(tpath))
        for k_, r_ in roofs.items():
            v_ = tr.get("dram_bytes_per_step", {}).get(k_)
            r_["traffic"] = v_ / max(B, 1) if v_ else None
            r_["traffic_note"] = "ncu dram__bytes_read+write per step (" + tr["source"] + ")"
    dom = ["condense", "factor", "solve"][int(np.argmax(ph_mean))]
    if dom == "factor" and "factor_large" in roofs and roofs["factor_large"]["time_share"] > 0.5:
        dom = "factor_large"     # the dominant KERNEL is the large-supernode DMMA kernel
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": value,
           "higher_is_better": False, "scaling": "strong" if batched else "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, synth/)",
           "config": config_of(args, inst, world),
           "analysis": {"nnzK": int(S.info["nnzK"]), "nnzL": int(S.info["nnzL"]),
                        "flops": S.info["flops"], "flops_large": S.info["flops_huge"],
                        "nsuper": S.info["nsuper"], "tree_height": S.info["tree_height"],
                        "max_front": S.info["max_front"], "analyze_ms": S.info["analyze_ms"],
                        "order_ms": S.info["order_ms"], "batch_per_gpu": B},
           "phases_ms": {n_: float(v_) for n_, v_ in zip(["condense", "factor", "solve"], ph_mean)},
           "factor_split_ms": {"small_big": float(fl_ms[0]), "large": float(fl_ms[1])},
           "instances_per_s": (C5_TOTAL if batched else world) / (value * 1e-3),
           "refine_iters": info["refine_iters"], "cg_iters": info["cg_iters"],
           **({"krylov_iters_total": krylov_total} if hykkt else {}),
           "bwd_err": info["bwd_err"], "wall_s_timed": t_wall,
           "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
           "gpu_launches": launches,
           "roofline": dict(roofs[dom], phase=dom),
           "roofline_phases": roofs,
           "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        ob = oracle_baseline(args, inst, args.cpu_sample_s, threads if batched else 1)
        if batched:
            val = ob["parallel"]["ms_per_instance"] * C5_TOTAL
            cores = ob["parallel"]["threads"]
            sample = (f"{ob['parallel']['instances']} C5 instances, one per thread on {cores} threads "
                      f"({ob['parallel']['wall_s']:.1f} s), scaled to the 512-instance batch; "
                      f"single-thread: {ob['iters']} iterations of one instance")
        else:
            val, cores = ob["iter_ms"], 1
            sample = (f"{ob['iters']} oracle IPM iterations of one {args.workload} instance (condense + "
                      f"Cholesky + __float128-refined solve), ~{args.cpu_sample_s:.0f} s budget after "
                      f"the once-per-pattern oracle analysis")
        out["cpu_baseline"] = dict({"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": sample, "phases_ms_1thread": ob["phases_ms"],
                                    "analysis_ms": ob["analysis_ms"]}, **cpu_info())
    if rank == 0:
        print(json.dumps(out), flush=True)
    S.close()
    if dist:
        dist.destroy_process_group()


def relaunch(args):
    """`--gpus N` without a torchrun environment: run this script under torch.distributed.run."""
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(relaunch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
