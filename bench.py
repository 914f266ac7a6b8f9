#!/usr/bin/env python
"""Benchmark of the B200 global-registration path (BASELINE.json configs[1]).

Workload B1: register_global on a 640x480 depth-frame pair of
the synthetic room scene (~307k points per cloud), 1,000,000 RANSAC
hypotheses, seed 1. One step = one pass of the hypothesis path (sampling ->
pre-rejection -> Kabsch -> scoring -> arg-best) over the full hypothesis
range, sharded contiguously over ranks, plus the cross-rank record exchange.

  value  candidate x point evaluations per second (W_ref / device time),
         context resident in HBM, L2 flushed before every timed step.
  e2e    the same metric through the public API from pinned host clouds:
         prepare_registration + run + exchange + merge, every step.

`python bench.py --impl reference` times the reference itself on the host
cores: its own registration sources compiled unmodified into oracle/_ref
(oracle/Makefile.ref, Eigen/doctest shim; OpenMP on every host thread), or the
oracle restatement where that build is absent, on the same workload and metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate×point evals/sec"
UNIT = "evals/s"
PAPER_MS_PER_REGISTRATION = 20.50  # PAPER.md:161 (Titan X Pascal, redwood pairs) -- context only


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--hypotheses", type=int, default=1_000_000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the config D (ICP) and E (verification) legs")
    ap.add_argument("--verify-pairs", type=int, default=256)
    return ap.parse_args()


def workload_config(args, ns_raw, nt_raw, ns=None, nt=None):
    cfg = {
        "workload": "B1: register_global on a 640x480 room-scene depth-frame pair "
                    f"(make_room_scene(1,6), orbit frames 0/6), H={args.hypotheses:,} hypotheses, seed {args.seed}",
        "source_points": ns_raw, "target_points": nt_raw,
        "hypotheses": args.hypotheses, "leaf": 0.05, "d_max": 0.075,
        "l2": "flushed before every timed step (256 MiB device write)",
        "parallelism": f"hypotheses sharded contiguously over {args.gpus} rank(s) (one process per GPU), one NCCL "
                       "all-reduce of the rank records inside the library (lk_reg_run_exchange)",
    }
    if ns is not None:
        cfg["source_downsampled"] = ns
        cfg["target_downsampled"] = nt
    return cfg


def make_fixture():
    from paper_1801_01572_b200 import synth
    return synth.depth_frame_pair(seed=1, boxes=6)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def onchip_peaks():
    """The ceilings of an L2-resident gather (tools/peaks.cu, run on this pool's
    B200s, committed as profiles/peaks.json): L2 random 32-B sector gather GB/s
    (best working set), FP32 FMA TFLOP/s, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks.json")) as f:
            p = json.load(f)
        l2 = max(x["gbs"] for x in p["l2_random_sector"])
        return {"l2_random_gbs": l2, "l2_stream_gbs": p["l2_stream"]["gbs"], "smem_gbs": p["smem"]["gbs"],
                "fp32_tflops": p["fp32_fma"]["tflops"], "fp64_tflops": p["fp64_fma"]["tflops"]}
    except Exception:
        return None


def ncu_roofline(kernels, bound):
    """Roofline of an extras leg's dominant kernels from the committed ncu
    capture (profiles/ncu_kernels.json; cold-cache, serialised launches):
    bound "l2_gather" = L2 sectors x 32 B / kernel time against the measured
    random-sector rate; bound "issue" = warp instructions / kernel time
    against 4 per SM per cycle at the measured clock."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_kernels.json")) as f:
            k = json.load(f)
        oc = onchip_peaks() or {}
        t = sum(k[n]["gpu__time_duration.sum"] for n in kernels) * 1e-9
        if bound == "l2_gather":
            achieved = sum(k[n]["lts__t_sectors.sum"] for n in kernels) * 32 / t / 1e9
            peak, unit = oc.get("l2_random_gbs"), "GB/s"
        else:
            achieved = sum(k[n]["smsp__inst_executed.sum"] for n in kernels) / t / 1e9
            peak, unit = 148 * 4 * 1.965, "G warp-instructions/s"
        dram = sum(k[n]["dram__bytes_read.sum"] + k[n]["dram__bytes_write.sum"] for n in kernels)
        return {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                "frac": achieved / peak if peak else None, "traffic": dram / max(1, len(kernels)),
                "kernel": "+".join(kernels), "kernel_ms_ncu": t * 1e3,
                "source": "profiles/ncu_kernels.json (ncu --metrics, cold-cache serialised launches)"}
    except Exception as e:
        return {"unavailable": str(e)[:120]}


def ncu_traffic(kernels):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernels`
    from the committed ncu --set full capture, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)["dram_bytes_per_launch"]
        return float(sum(t[k] for k in kernels))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout=5.0):
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.05)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


# ------------------------------------------------------------------ CPU
def _ref_module():
    """oracle/_ref (the reference's own sources, prebuilt) when present, else None."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref as RF
    return RF if os.path.exists(RF.LIB_PATH) else None


_W_REF = {}


def oracle_work(pair, hypotheses, seed):
    """The oracle's run of the workload: its work counters (W_ref = the points
    the reference loop visits, o / k / h of SURVEY.md 8d) are the metric's
    numerator; the reference does not count them."""
    key = (id(pair), hypotheses, seed)
    if key not in _W_REF:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        p = O.params(hypothesis_count=hypotheses, seed=seed, threads=os.cpu_count() or 0)
        ctx = O.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                pair.target.normals, p)
        res, st = ctx.run(p)
        _W_REF[key] = dict(stats=st, result=res, ns=ctx.ns, nt=ctx.nt)
    return _W_REF[key]


def cpu_reference_registration(pair, hypotheses, seed, budget_s=12.0, min_reps=1, max_reps=8):
    """The reference on the host cores: register_global's prepare + run_hypotheses
    from oracle/_ref (OpenMP schedule(dynamic,256), all threads), or the oracle
    restatement when _ref is absent. Repeats full registrations until ~budget_s
    of CPU work; returns the best repetition (kind "reference" or "port")."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    RF = _ref_module()
    mod, kind = (RF, "reference") if RF is not None else (O, "port")
    p = O.params(hypothesis_count=hypotheses, seed=seed, threads=os.cpu_count() or 0)
    work = oracle_work(pair, hypotheses, seed)
    best = None
    t_start = time.perf_counter()
    reps = 0
    while reps < min_reps or (time.perf_counter() - t_start < budget_s and reps < max_reps):
        t0 = time.perf_counter()
        ctx = mod.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                  pair.target.normals, p)
        t1 = time.perf_counter()
        res, st = ctx.run(p)
        t2 = time.perf_counter()
        rec = dict(prepare_s=t1 - t0, run_s=t2 - t1, stats=dict(work["stats"]), result=res, ns=ctx.ns, nt=ctx.nt,
                   kind=kind, parity=(res.hypothesis_index == work["result"].hypothesis_index))
        if best is None or rec["prepare_s"] + rec["run_s"] < best["prepare_s"] + best["run_s"]:
            best = rec
        reps += 1
    best["reps"] = reps
    return best


def work_shape(stats):
    """o, k, h of SURVEY.md 8d from the oracle's counters, and bytes / flops per eval."""
    w = max(stats["w_ref"], 1)
    o = stats["near_occupied"] / w
    k = stats["slots_scanned"] / w
    h = stats["nn_hits"] / w
    return dict(o=o, k=k, h=h, bytes_per_eval=1 + 72 * o + 12 * k + 12 * h, flop_per_eval=24 + 8 * k + 21 * h)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0  # N>1: rank 0 alone runs the host baseline
    # torchrun sets OMP_NUM_THREADS=1 per rank; the baseline uses every host thread
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    pair = make_fixture()
    threads = os.cpu_count()
    times, wref = [], None
    for step in range(args.warmup + args.steps):
        rec = cpu_reference_registration(pair, args.hypotheses, args.seed, budget_s=0.0)
        if step >= args.warmup:
            times.append(rec)
        wref = rec["stats"]["w_ref"]
    run_s = sum(r["run_s"] for r in times) / len(times)
    reg_s = sum(r["prepare_s"] + r["run_s"] for r in times) / len(times)
    value = wref / run_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": run_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, pair.source.size(), pair.target.size(), times[0]["ns"], times[0]["nt"]),
        "ms_per_registration": reg_s * 1e3,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": times[0]["kind"],
                         "sample": f"full B1 registration per step (prepare + {args.hypotheses:,} hypotheses), "
                                   + ("the reference's own sources (oracle/_ref, -O3, Eigen shim)"
                                      if times[0]["kind"] == "reference" else "oracle restatement")
                                   + ", OpenMP dynamic,256 on all host threads; W_ref from the oracle's counters"},
        "e2e": {"value": wref / reg_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "ms_per_registration": reg_s * 1e3},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ extras
def _pinned_cloud(c):
    """The cloud's arrays copied into pinned host memory (the H2D inside the
    timed calls then runs at full PCIe rate), and the tensors that own it."""
    import torch
    import paper_1801_01572_b200 as lk
    tp = torch.from_numpy(np.ascontiguousarray(c.positions)).pin_memory()
    tn = torch.from_numpy(np.ascontiguousarray(c.normals)).pin_memory() if c.normals is not None else None
    return lk.PointCloud(tp.numpy(), tn.numpy() if tn is not None else None), (tp, tn)


def _pool_map(fn, items):
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:  # ctypes calls release the GIL
        return list(ex.map(fn, items))


def bench_icp(args):
    """Config D: register_global (H = 10^6) on the 2.4M-point
    submap pair, then ICP point-to-plane on the full clouds from the global
    result, both through the public API from pinned host buffers (uploads,
    prepare, grids and every ICP iteration inside the timing). CPU baseline:
    the oracle's register_global on the same pair and one oracle ICP
    iteration, scaled by the device's iteration count."""
    import numpy as np
    import paper_1801_01572_b200 as lk
    from paper_1801_01572_b200 import synth
    pair = synth.submap_pair()
    src, keep_s = _pinned_cloud(pair.source)
    tgt, keep_t = _pinned_cloud(pair.target)
    params = lk.RegistrationParams(hypothesis_count=1_000_000, seed=1)
    ip = lk.IcpParams(max_correspondence_distance=0.05, max_iterations=30, convergence_eps=1e-10)
    reg = lk.register_global(src, tgt, params)  # warm-up
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        reg = lk.register_global(src, tgt, params)
        t1 = time.perf_counter()
        r = lk.icp_point_to_plane(src, tgt, reg.transform, ip)
        t2 = time.perf_counter()
        if best is None or (t2 - t0) < best[0] + best[1]:
            best = (t1 - t0, t2 - t1)

    def err(T):
        R = pair.truth.rotation.T @ T.rotation
        return (float(np.degrees(np.arccos(np.clip((np.trace(R) - 1) / 2, -1, 1)))),
                float(np.linalg.norm(T.translation - pair.truth.translation)))
    evaluated = len(r.history)
    out = {"workload": "D: submap_pair(seed 2, 8 views x 640x480 per submap, no downsample): register_global "
                       "(H = 10^6, seed 1), then ICP point-to-plane (d = 0.05 m) from its result",
           "source_points": pair.source.size(), "target_points": pair.target.size(),
           "ms_register_global": 1e3 * best[0], "ms_icp": 1e3 * best[1], "ms_total": 1e3 * (best[0] + best[1]),
           "global_error_deg_m": err(reg.transform), "icp_error_deg_m": err(r.transform),
           "icp_iterations": r.iterations, "icp_converged": r.converged, "icp_correspondences": r.correspondences,
           "icp_rmse": r.rmse, "icp_ms_per_iteration": 1e3 * best[1] / max(evaluated, 1),
           "icp_point_iterations_per_s": pair.source.size() * evaluated / best[1],
           "h2d_bytes": 2 * 48 * (pair.source.size() + pair.target.size()),
           "timing": "wall clock of lk_register_global + lk_icp_point_to_plane from pinned host buffers, best of 3",
           "roofline": ncu_roofline(["k_icp_nn"], "issue")}
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        t0 = time.perf_counter()
        p = O.params(hypothesis_count=1_000_000, seed=1, threads=os.cpu_count() or 0)
        ctx = O.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                pair.target.normals, p)
        res, _ = ctx.run(p)
        cpu_reg = time.perf_counter() - t0
        t0 = time.perf_counter()
        R1, t1_, res1, h1 = O.icp_point_to_plane(pair.source.positions, pair.target.positions, pair.target.normals,
                                                 reg.transform.rotation, reg.transform.translation, 0.05, 1, 0.0)
        cpu_it = time.perf_counter() - t0
        out["cpu_baseline"] = {"kind": "port", "cores": os.cpu_count(),
                               "sample": "the oracle's register_global on the pair, and one oracle ICP iteration "
                                         "(grid build + accumulation + solve) scaled by the device's iteration count",
                               "ms_register_global": 1e3 * cpu_reg,
                               "ms_icp_extrapolated": 1e3 * cpu_it * evaluated,
                               "parity": {"hypothesis_index": bool(res.found and
                                                                   res.hypothesis_index == reg.hypothesis_index),
                                          "icp_first_iteration": bool(h1[0, 0] == r.history[0, 0]
                                                                      and h1[0, 1] == r.history[0, 1])}}
    return out


def bench_b2(args):
    """Config B2: explicit candidate scoring on the full
    resolution pair (~307k points each, no downsample), a rotation x
    translation lattice around the truth (1 deg / 1 cm), evaluate_against_grid
    semantics with the miss budget; a bounded sample of the 10^6-candidate
    lattice (throughput and roofline only). The dense target's EvalGrid
    neighbour comes from the ring grid."""
    import paper_1801_01572_b200 as lk
    from paper_1801_01572_b200 import synth
    pair = synth.depth_frame_pair()
    rt, _ = synth.lattice_candidates(pair.truth, math.pi / 180.0, 0.01, 2, 2)  # 125 x 125 = 15,625 candidates
    params = lk.RegistrationParams()
    grid = lk.build_eval_grid(pair.target, params.d_max)
    lk.score_candidates(grid, pair.source, rt[:2048], params, early_exit=True)  # warm-up
    times = []
    for _ in range(2):
        t0 = time.perf_counter()
        sc = lk.score_candidates(grid, pair.source, rt, params, early_exit=True)
        times.append(time.perf_counter() - t0)
    dt = min(times)
    evals = rt.shape[0] * pair.source.size()
    out = {"workload": "B2: depth_frame_pair at full resolution, lattice_candidates(truth, 1 deg, 1 cm, "
                       "rot +-2, trans +-2) = 15,625 of the 10^6-candidate lattice, early exit on, best of 2",
           "candidates": int(rt.shape[0]), "source_points": pair.source.size(), "target_points": pair.target.size(),
           "evals": evals, "ms": 1e3 * dt, "evals_per_s": evals / dt, "qualified": sc.qualified,
           "timing": "wall clock of lk_score_candidates (candidates H2D, scoring, per-candidate results D2H)",
           "full_lattice": "tools/b2_full.py: all 10^6 candidates device-side, profiles/r02_b2_full.json",
           "roofline": ncu_roofline(["k_score_list_ring"], "issue")}
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        sample = rt[:4]
        t0 = time.perf_counter()
        O.score_candidates(pair.source.positions, pair.source.normals, pair.target.positions, pair.target.normals,
                           sample, 0, 1, 0.0, O.params())
        cpu = time.perf_counter() - t0
        out["cpu_baseline"] = {"kind": "port", "cores": os.cpu_count(),
                               "sample": "the oracle on the first 4 candidates (EvalGrid build included)",
                               "evals_per_s": sample.shape[0] * pair.source.size() / cpu}
    return out


def bench_config_a(args):
    """configs[0]: the ~10k-point scatter-scene surface
    pair (density 150, noise 0.005): all 9,261 lattice candidates scored with
    evaluate_hypothesis semantics (SearchGrid cell 0.075, no early exit), and
    register_global H = 10^4 seed 1, through the public API from host arrays.
    Parity against the committed reference golden file (oracle/_ref output)."""
    import paper_1801_01572_b200 as lk
    from paper_1801_01572_b200 import synth
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_golden.json")))
    pair = synth.surface_pair(1, density=150.0)
    rt, ti = synth.lattice_candidates(pair.truth)
    params = lk.RegistrationParams()
    grid = lk.build_grid(pair.target, 0.075)
    lk.score_candidates(grid, pair.source, rt[:64], params)  # warm-up
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        sc = lk.score_candidates(grid, pair.source, rt, params)
        times.append(time.perf_counter() - t0)
    lat_s = min(times)
    evals = rt.shape[0] * pair.source.size()
    rp = lk.RegistrationParams(hypothesis_count=10_000, seed=1)
    lk.register_global(pair.source, pair.target, rp)  # warm-up
    rtimes, st = [], lk.HypothesisStats()
    for _ in range(5):
        t0 = time.perf_counter()
        res = lk.register_global(pair.source, pair.target, rp, st)
        rtimes.append(time.perf_counter() - t0)
    out = {"workload": "A: surface_pair(make_scatter_scene(1), density 150, noise 0.005): 9,261-candidate lattice "
                       "(2 deg / 2 cm around truth, evaluate_hypothesis semantics) + register_global H=1e4 seed 1",
           "source_points": pair.source.size(), "target_points": pair.target.size(),
           "lattice_candidates": int(rt.shape[0]), "lattice_evals": evals, "lattice_ms": 1e3 * lat_s,
           "lattice_evals_per_s": evals / lat_s,
           "register_ms": 1e3 * min(rtimes), "register_index": res.hypothesis_index if res else -1,
           "parity_vs_reference_golden": {
               "lattice_inliers": sc.inliers.tolist() == g["a_lattice"]["inliers"],
               "register_index": bool(res and res.hypothesis_index == g["a_register"]["index"]),
               "register_stats": {k: getattr(st, k) for k in ("sampled", "prerejected", "degenerate", "evaluated",
                                                              "qualified")} == g["a_register"]["stats"]},
           "timing": "wall clock of lk_score_candidates (candidates H2D, scoring, per-candidate results D2H) and of "
                     "lk_register_global from pageable numpy arrays, best of 5"}
    if not args.no_cpu_baseline:
        RF = _ref_module()
        if RF is not None:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as O
            op = O.params()
            sample = list(range(0, rt.shape[0], 97))

            def one(k):
                return RF.evaluate_hypothesis(rt[k, :9].reshape(3, 3), rt[k, 9:], pair.source.positions,
                                              pair.source.normals, pair.target.positions, pair.target.normals,
                                              0.075, op)
            t0 = time.perf_counter()
            _pool_map(one, sample)
            cpu_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            RF.register_global(pair.source.positions, pair.source.normals, pair.target.positions,
                               pair.target.normals, O.params(hypothesis_count=10_000, seed=1,
                                                             threads=os.cpu_count() or 0))
            cpu_reg = time.perf_counter() - t0
            out["cpu_baseline"] = {"kind": "reference", "cores": os.cpu_count(),
                                   "sample": f"oracle/_ref evaluate_hypothesis on {len(sample)} of the lattice "
                                             "candidates (one per host thread), and its register_global",
                                   "lattice_evals_per_s": len(sample) * pair.source.size() / cpu_s,
                                   "register_ms": 1e3 * cpu_reg}
    return out


def bench_propose_loops(args):
    """Row f2, propose_loops (fragments.cpp:61-109): 32 fragments
    of 4,000 random points in a 1 m cube under small random poses (every
    pair overlaps), all (i, j <= i - 2) pairs = 465 pair overlaps of 4,000
    queries each, one lk_propose_loops call from host arrays. Parity: the
    proposals (i, j, overlap bits) against the reference's own propose_loops
    (oracle/_ref) on the same input, which is also the CPU baseline."""
    import paper_1801_01572_b200 as lk
    from paper_1801_01572_b200 import synth
    F, npts = 32, 4000
    frags = [synth.random_cloud(npts, 100 + f, 0, -0.5, 0.5) for f in range(F)]
    poses = [synth.random_transform(200 + f, 1, 0.3, 0.3) for f in range(F)]
    lp = lk.LoopParams(overlap_radius=0.05, min_overlap=0.2)
    lk.propose_loops(frags, poses, [], lp)  # warm-up
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        got = lk.propose_loops(frags, poses, [], lp)
        times.append(time.perf_counter() - t0)
    dt = min(times)
    pairs = (F - 1) * (F - 2) // 2
    out = {"workload": f"propose_loops: {F} fragments x {npts:,} random points (1 m cube), small random poses, "
                       f"overlap radius 0.05, min_overlap 0.2: {pairs} pair overlaps",
           "fragments": F, "points_per_fragment": npts, "pairs": pairs, "proposals": len(got), "ms": 1e3 * dt,
           "pairs_per_s": pairs / dt, "queries_per_s": pairs * npts / dt,
           "timing": "wall clock of lk_propose_loops from host arrays (H2D, posed ring grids, all pairs, host "
                     "filter and sort), best of 3"}
    if not args.no_cpu_baseline:
        RF = _ref_module()
        if RF is not None:
            t0 = time.perf_counter()
            ref = RF.propose_loops([f.positions for f in frags], [(T.rotation, T.translation) for T in poses], (),
                                   0.05, 0.2)
            cpu = time.perf_counter() - t0
            out["parity_vs_reference"] = [(p.i, p.j, float(p.overlap).hex()) for p in got] == \
                [(i, j, float(v).hex()) for i, j, v in ref]
            out["cpu_baseline"] = {"kind": "reference", "cores": 1,
                                   "sample": "oracle/_ref propose_loops on the same input (the reference loop, one "
                                             "thread)", "ms": 1e3 * cpu, "pairs_per_s": pairs / cpu}
    return out


def bench_verification(args):
    """Config E: loop verification of synth_registration_pair
    seeds 1..K with their truths as measurements: edge_info(Q, P, I, truth,
    0.05), the propose_loops overlap within 0.1 m and evaluate_hypothesis(truth)
    per pair, one lk_verify_batch call from host buffers."""
    import paper_1801_01572_b200 as lk
    from paper_1801_01572_b200 import synth
    K = args.verify_pairs
    pairs = _pool_map(synth.synth_registration_pair, range(1, K + 1))
    pinned = [(_pinned_cloud(p.target), _pinned_cloud(p.source)) for p in pairs]
    Q = [q for (q, _), _ in pinned]
    P = [s for _, (s, _) in pinned]
    I = [lk.RigidTransform() for _ in pairs]
    T = [p.truth for p in pairs]
    vp = lk.VerifyParams()
    lk.verify_batch(Q, P, I, T, T, vp)  # warm-up
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        out = lk.verify_batch(Q, P, I, T, T, vp)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * min(times)
    npts = sum(p.source.size() + p.target.size() for p in pairs)
    res = {"workload": f"E: synth_registration_pair(1..{K}), measurement = truth; edge_info eps 0.05, overlap "
                       "r 0.1, evaluate_hypothesis d_max 0.075 / 30 deg",
           "pairs": K, "points": npts, "ms_per_batch": ms, "pairs_per_s": K / (ms / 1e3),
           "mean_overlap": float(np.mean([o.overlap for o in out])),
           "mean_inlier_ratio": float(np.mean([o.inlier_ratio for o in out])),
           "h2d_bytes": 48 * npts,
           "timing": "wall clock of lk_verify_batch from pinned host buffers (H2D, 3K ring grids, queries, "
                     "sums), best of 5",
           "roofline": ncu_roofline(["k_verify_src", "k_verify_edge"], "l2_gather")}
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        op = O.params()
        sample = pairs[:32]

        def one(p):
            try:
                O.edge_info(p.target.positions, p.source.positions, np.eye(3), np.zeros(3), p.truth.rotation,
                            p.truth.translation, 0.05)
            except O.OracleError:
                pass
            h = O.overlap_hits(p.source.positions, p.truth.rotation, p.truth.translation, p.target.positions,
                               np.eye(3), np.zeros(3), 0.1)
            e = O.evaluate_hypothesis(p.truth.rotation, p.truth.translation, p.source.positions, p.source.normals,
                                      p.target.positions, p.target.normals, 0.075, op)
            return h, e
        t0 = time.perf_counter()
        chk = _pool_map(one, sample)
        cpu_s = time.perf_counter() - t0
        res["cpu_baseline"] = {"kind": "port", "cores": os.cpu_count(),
                               "sample": f"the oracle on the first {len(sample)} pairs, one pair per host thread",
                               "pairs_per_s": len(sample) / cpu_s,
                               "parity": all(h == o.overlap_hits and e[2] == o.inliers and e[1] == o.fitness
                                             for (h, e), o in zip(chk, out[:len(sample)]))}
    return res


# ------------------------------------------------------------------ GPU
def count_kernel_launches(step, torch):
    """Kernels of this library launched by one (untimed) step, counted from a
    CUPTI trace (torch.profiler); library kernels live in namespace lkk."""
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        import re
        names = [e.name for e in prof.events() if "lkk::" in e.name]
        per = {}
        for n in names:
            m = re.search(r"\b(k_\w+)", n)
            k = m.group(1) if m else n[:60]
            per[k] = per.get(k, 0) + 1
        return len(names), per
    except Exception as e:  # profiler unavailable: report it, do not guess
        return None, {"error": str(e)[:200]}


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1801_01572_b200 as lk
    from paper_1801_01572_b200 import abi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: LK_BENCH_ONE_DEVICE=1 runs every rank on cuda:0 over gloo
    # (exercises the multi-rank path on a single-GPU box; not a bench mode)
    one_dev = os.environ.get("LK_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    # a dedicated stream: the library launches on it and the CUDA events are
    # recorded on it (torch's default stream is the legacy NULL stream)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    pair = make_fixture()
    H = args.hypotheses
    params = lk.RegistrationParams(hypothesis_count=H, seed=args.seed, device=local)
    begin, end = rank * H // world, (rank + 1) * H // world

    # pinned host copies of the raw clouds (inputs of the e2e leg)
    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t, t.numpy()
    keep = []
    clouds = []
    for c in (pair.source, pair.target):
        tp, p_np = pinned(c.positions)
        tn, n_np = pinned(c.normals)
        keep += [tp, tn]
        clouds.append(lk.PointCloud(p_np, n_np))
    src_h, tgt_h = clouds

    words = abi.C.sizeof(abi.lk_reg_record) // 8
    xbuf = torch.zeros(world * words, dtype=torch.int64, device=dev)
    slot_ptr = xbuf.data_ptr() + rank * words * 8
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # ---- device-resident leg
    ctx = lk.prepare_registration(src_h, tgt_h, params)
    ctx.set_stream(stream.cuda_stream)
    # N > 1: the library's own exchange -- rank 0's NCCL unique id goes to every
    # rank, each context joins the communicator, and lk_reg_run_exchange runs
    # the rank's share and the ncclAllReduce of the rank records on the
    # context stream (include/loopkit_b200.h). The one-device test hook (every
    # rank on cuda:0, gloo) cannot host an NCCL communicator: it exchanges
    # through torch.
    lib_exchange = world > 1 and not one_dev
    if lib_exchange:
        box = [lk.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ctx.attach_comm(box[0], world, rank)

    def step():
        if lib_exchange:
            ctx.run_exchange(params, xbuf.data_ptr())
            return
        xbuf.zero_()
        lk.run_hypotheses_range(ctx, params, begin, end, slot_ptr)
        if world > 1:
            dist.all_reduce(xbuf)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    ctx.kernel_times(reset=True)
    ctx.set_profiling(True)
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
        clocks.wait_first()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()  # L2 flush, outside the timed interval
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clock_info = clocks.stop() if rank == 0 else None
    ctx.set_profiling(False)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    launches_per_step, launch_kinds = count_kernel_launches(step, torch)
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    total_ms = float(total_ms.item())
    kt, runs = ctx.kernel_times()
    ph, _ = ctx.phase_times()
    recs = lk.records_from_bytes(xbuf.cpu().numpy())
    mstats = lk.HypothesisStats()
    merged = lk.merge_records(recs, ctx.n_source, mstats)
    w_step = mstats.w_ref  # all ranks, one step
    value = w_step * args.steps / (total_ms / 1e3)

    # ---- end-to-end leg through the public API from pinned host memory
    e2e_steps = args.e2e_steps or 20
    e2e_warm = max(3, args.warmup)  # untimed: the first calls grow the memory pool and pinned staging
    e2e_times = []
    h2d = d2h = 0
    rec_bytes = abi.C.sizeof(abi.lk_reg_record)
    for k in range(e2e_steps + e2e_warm):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            # one process, one GPU: the drop-in call itself (lk_register_global:
            # prepare, hypotheses, record readback, merge)
            res = lk.register_global(src_h, tgt_h, params)
            out_bytes = rec_bytes
        else:
            c2 = lk.prepare_registration(src_h, tgt_h, params)
            c2.set_stream(stream.cuda_stream)
            xbuf.zero_()
            lk.run_hypotheses_range(c2, params, begin, end, slot_ptr)
            dist.all_reduce(xbuf)
            host = xbuf.cpu().numpy()
            res = lk.merge_records(lk.records_from_bytes(host), c2.n_source)
            out_bytes = host.nbytes
            c2.close()
        t1 = time.perf_counter()
        if k >= e2e_warm:
            e2e_times.append(t1 - t0)
        # bytes copied this step: the raw clouds (positions + normals) in; out,
        # the record(s) plus the library's control readbacks per cloud side
        # (voxel count + normal check 8 B, FPFH staging head: 20 B of counts,
        # 2048 acos records of 32 B and 64 theta-edge records of 96 B, cloud
        # stats 16 B) and the EvalGrid's bounds and block total (28 B); acos
        # records beyond the staged 2048 add 32 B each (not counted)
        h2d = 48 * (src_h.size() + tgt_h.size())
        d2h = 2 * (8 + 20 + 2048 * 32 + 64 * 96 + 16) + 28 + out_bytes
    e2e_s = torch.tensor([statistics.mean(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s.item())

    # the same leg from pageable host arrays, as the drop-in register_global
    # receives them (std::vector / numpy; registration.hpp:121-124)
    src_p = lk.PointCloud(np.array(pair.source.positions), np.array(pair.source.normals))
    tgt_p = lk.PointCloud(np.array(pair.target.positions), np.array(pair.target.normals))
    pg_times = []
    for k in range(e2e_steps + e2e_warm):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            lk.register_global(src_p, tgt_p, params)
        else:
            c3 = lk.prepare_registration(src_p, tgt_p, params)
            c3.set_stream(stream.cuda_stream)
            xbuf.zero_()
            lk.run_hypotheses_range(c3, params, begin, end, slot_ptr)
            dist.all_reduce(xbuf)
            lk.merge_records(lk.records_from_bytes(xbuf.cpu().numpy()), c3.n_source)
            c3.close()
        t1 = time.perf_counter()
        if k >= e2e_warm:
            pg_times.append(t1 - t0)
    pg_s = torch.tensor([statistics.mean(pg_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(pg_s, op=dist.ReduceOp.MAX)
    pg_s = float(pg_s.item())

    if rank == 0:
        hbm_peak, peak_kind = peaks()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, pair.source.size(), pair.target.size(), ctx.n_source, ctx.n_target),
            "found": merged is not None,
            "hypothesis_index": merged.hypothesis_index if merged else -1,
            "stats_per_step": {k: getattr(mstats, k) for k in ("sampled", "prerejected", "degenerate", "evaluated",
                                                              "qualified", "w_ref", "evals_executed")},
            "kernel_ms_per_step": {k: v / max(runs, 1) for k, v in ph.items()},
            "e2e": {"value": w_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_registration": e2e_s * 1e3,
                    "steps": len(e2e_times), "statistic": "mean",
                    "note": ("lk_register_global from page-locked host clouds: H2D of the raw clouds, voxel "
                             "downsample, FPFH, feature match, EvalGrid, hypotheses, record readback, merge"
                             if world == 1 else
                             "prepare_registration from page-locked host clouds + the rank's hypotheses + the "
                             "record all-reduce + merge")},
            "e2e_pageable": {"value": w_step / pg_s, "unit": UNIT, "ms_per_registration": pg_s * 1e3,
                             "h2d_bytes_per_step": int(h2d),
                             "note": "the e2e leg from pageable numpy arrays (what a drop-in register_global "
                                     "caller passes), H2D staged by the driver"},
            "paper_ms_per_registration": PAPER_MS_PER_REGISTRATION,
            "gpu_launches": launches_per_step * args.steps if launches_per_step is not None else None,
            "gpu_launches_per_step": launch_kinds,
            "clocks": clock_info,
        }
        # roofline of the scoring kernel (every candidate x point evaluation
        # happens there), algorithmic bytes per SURVEY.md 8d, event-timed on
        # the launch stream
        score_kernels = [k for k in ph if k not in ("k_hyp_sample", "k_kabsch")]
        score_ms = sum(ph[k] for k in score_kernels) / max(runs, 1)
        shape = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_reference_registration(pair, H, args.seed)
            shape = work_shape(cpu["stats"])
            line["cpu_baseline"] = {
                "value": cpu["stats"]["w_ref"] / cpu["run_s"], "unit": UNIT, "cores": os.cpu_count(),
                "kind": cpu["kind"],
                "sample": f"{cpu['reps']} full B1 registration(s) on "
                          + ("the reference's own sources (oracle/_ref)" if cpu["kind"] == "reference"
                             else "the oracle") + f" (prepare + {H:,} hypotheses); "
                          f"best {1e3 * (cpu['prepare_s'] + cpu['run_s']):.1f} ms/registration, "
                          f"hypothesis stage {1e3 * cpu['run_s']:.1f} ms; W_ref from the oracle's counters",
                "ms_per_registration": 1e3 * (cpu["prepare_s"] + cpu["run_s"]),
                "parity": {"reference_index": cpu["result"].hypothesis_index,
                           "b200_index": merged.hypothesis_index if merged else -1,
                           "oracle_w_ref": cpu["stats"]["w_ref"], "b200_w_ref": w_step},
            }
        if shape is None:
            shape = {"o": None, "k": None, "h": None, "bytes_per_eval": None}
        evals_per_launch = mstats.evals_executed / max(world, 1)
        if shape["bytes_per_eval"] and score_ms > 0:
            achieved = evals_per_launch * shape["bytes_per_eval"] / (score_ms / 1e3) / 1e9
            flops = evals_per_launch * shape["flop_per_eval"] / (score_ms / 1e3) / 1e12
            traffic = ncu_traffic(score_kernels)
            oc = onchip_peaks()
            if oc:
                peak, unit, kind = oc["l2_random_gbs"], "GB/s", "measured (tools/peaks.cu -> profiles/peaks.json)"
            else:
                peak, unit, kind = hbm_peak, "GB/s", peak_kind + " HBM (profiles/peaks.json absent)"
            line["roofline"] = {"bound": "l2_gather" if oc else "hbm", "achieved": achieved, "peak": peak,
                                "unit": unit, "frac": achieved / peak, "traffic": traffic,
                                "kernel": "+".join(score_kernels), "peak_kind": kind,
                                "evals_per_launch": evals_per_launch, "kernel_ms": score_ms, "work_shape": shape,
                                "fp32": {"achieved_tflops": flops,
                                         "peak_tflops": oc["fp32_tflops"] if oc else None,
                                         "frac": flops / oc["fp32_tflops"] if oc else None},
                                "hbm": {"dram_gbs": traffic / (score_ms / 1e3) / 1e9 if traffic else None,
                                        "peak_gbs": hbm_peak,
                                        "frac": traffic / (score_ms / 1e3) / 1e9 / hbm_peak if traffic else None},
                                "note": "achieved = evals executed per step x algorithmic on-chip bytes/eval "
                                        "(1+72o+12k+12h, SURVEY.md 8d) / event time of the scoring kernel on its "
                                        "launch stream; peak = the measured L2 random 32-B sector gather rate "
                                        "(the working set is L2-resident: DRAM traffic per launch is `traffic`, "
                                        "from the committed ncu capture profiles/ncu_traffic.json)"}
        if world == 1 and not args.no_extras:
            line["extras"] = {"config_A": bench_config_a(args), "icp_D": bench_icp(args),
                              "verification_E": bench_verification(args), "explicit_B2": bench_b2(args),
                              "propose_loops_F2": bench_propose_loops(args)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
