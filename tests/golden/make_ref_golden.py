"""Generates tests/golden/ref_golden.json from the REFERENCE's own code: the
reference sources compiled unmodified into oracle/_ref/liblk_ref.so
(oracle/Makefile.ref, Eigen/doctest shim in oracle/ref_shim/). These are
reference outputs, not oracle outputs: tests check the oracle (CPU) and the
B200 path (GPU, where /root/reference does not exist) against them.
Work counters the reference does not expose (W_ref) come from the oracle and
are marked "oracle_*".

    python tests/golden/make_ref_golden.py      # needs /root/reference (~3 min)
"""
import json
import math
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
import ref as RF  # noqa: E402

STATS = ("sampled", "prerejected", "degenerate", "evaluated", "qualified")


def hexd(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).reshape(-1)]


def csum(a):
    """bit-level checksum of an array (sum of its 64-bit words, mod 2^64)"""
    b = np.ascontiguousarray(a)
    pad = (-b.nbytes) % 8
    raw = np.frombuffer(b.tobytes() + b"\0" * pad, dtype=np.uint64)
    return int(raw.sum(dtype=np.uint64))


def result_dict(r, st):
    return dict(found=bool(r.found), index=int(r.hypothesis_index), inliers=int(r.inliers),
                ratio=float(r.inlier_ratio).hex(), fitness=float(r.fitness).hex(), R=hexd(r.R), t=hexd(r.t),
                stats={k: int(st[k]) for k in STATS})


def run_case(src, tgt, H, seed):
    p = O.params(hypothesis_count=H, seed=seed)
    ctx = RF.Context.prepare(src[0], src[1], tgt[0], tgt[1], p)
    c = ctx.get()
    r, st = ctx.run(p)
    d = result_dict(r, st)
    d.update(H=H, seed=seed, ns=ctx.ns, nt=ctx.nt, cache_sum=csum(c["cache"]), src_feat_sum=csum(c["src_feat"]),
             tgt_feat_sum=csum(c["tgt_feat"]), src_sum=csum(c["src"]), tgt_sum=csum(c["tgt"]))
    oc = O.Context.from_prepared(c["src"], c["src_n"], c["tgt"], c["tgt_n"], c["cache"], p.d_max)
    _, ost = oc.run(p)
    d["oracle_w_ref"] = int(ost["w_ref"])
    return d


def main():
    g = {"about": __doc__.strip().splitlines()[0],
         "shim": "oracle/ref_shim (Eigen 3.4 SSE2 order restated; see oracle/ref_shim/Eigen/Dense)"}
    # registration pairs (proj/src/synth.cpp:587-623) at the reference test's H / seeds
    runs = []
    for pair_seed in (1, 2):
        fx = RF.registration_pair(pair_seed)
        for seed, H in ((1, 20_000), (7, 20_000)):
            d = run_case(fx["source"], fx["target"], H, seed)
            d.update(pair=pair_seed, n_src=int(fx["source"][0].shape[0]), n_tgt=int(fx["target"][0].shape[0]),
                     raw_src_sum=csum(fx["source"][0]), raw_tgt_sum=csum(fx["target"][0]))
            runs.append(d)
    g["run_hypotheses"] = runs
    # B1 (configs[1]): the 640x480 room pair, H = 1e6, seed 1
    fx = RF.frame_pair()
    d = run_case(fx["source"], fx["target"], 1_000_000, 1)
    d.update(n_src=int(fx["source"][0].shape[0]), n_tgt=int(fx["target"][0].shape[0]),
             raw_src_sum=csum(fx["source"][0]), raw_tgt_sum=csum(fx["target"][0]))
    g["b1"] = d
    # config A (configs[0]): surface pair of make_scatter_scene(1), density 150 (|Q| ~ 10k)
    fx = RF.surface_pair(1, 150.0)
    src, tgt = fx["source"], fx["target"]
    d = run_case(src, tgt, 10_000, 1)
    d.update(density=150.0, n_src=int(src[0].shape[0]), n_tgt=int(tgt[0].shape[0]), raw_src_sum=csum(src[0]),
             raw_tgt_sum=csum(tgt[0]))
    g["a_register"] = d
    # config A explicit lattice: truth o transform_from_twist(delta), delta on
    # {-3..3} x 2 deg, {-1,0,1} x 0.02 m (lexicographic), evaluate_hypothesis
    # (registration.cpp:53-78) over build_grid(target, 0.075)
    Rt, tt = fx["truth"]
    step_r, step_m = 2.0 * math.pi / 180.0, 0.02
    cands = []
    for a in range(-3, 4):
        for b in range(-3, 4):
            for c in range(-3, 4):
                for x in (-1, 0, 1):
                    for y in (-1, 0, 1):
                        for z in (-1, 0, 1):
                            Rd, td = RF.transform_from_twist([a * step_r, b * step_r, c * step_r, x * step_m,
                                                              y * step_m, z * step_m])
                            cands.append(RF.compose(Rt, tt, Rd, td))
    p = O.params()
    ns = src[0].shape[0]

    def score(k):
        R, t = cands[k]
        return RF.evaluate_hypothesis(R, t, src[0], src[1], tgt[0], tgt[1], 0.075, p)

    with ThreadPoolExecutor(os.cpu_count()) as ex:
        scores = list(ex.map(score, range(len(cands))))
    g["a_lattice"] = {"seed": 1, "density": 150.0, "count": len(cands), "truth_index": 4630, "grid_cell": 0.075,
                      "cand_sum": csum(np.array([np.concatenate([R.reshape(9), t]) for R, t in cands])),
                      "inliers": [int(round(r * ns)) for r, _ in scores],
                      "fitness": [float(f).hex() for _, f in scores]}
    # config E: loop pairs synth_registration_pair(s), edge_info(Q, P, I, truth, 0.05)
    # (line_process.cpp:11-33) and evaluate_hypothesis(truth) (SearchGrid cell 0.075)
    e_pairs = []
    for s in (1, 3, 4, 5):
        fx = RF.registration_pair(s)
        (P, Pn), (Q, Qn) = fx["source"], fx["target"]
        R, t = fx["truth"]
        info, cnt = RF.edge_info(Q, P, np.eye(3), np.zeros(3), R, t, 0.05)
        ratio, fit = RF.evaluate_hypothesis(R, t, P, Pn, Q, Qn, 0.075, p)
        e_pairs.append(dict(seed=s, eps=0.05, pair_count=int(cnt), info=hexd(info), ratio=float(ratio).hex(),
                            fitness=float(fit).hex(), inliers=int(round(ratio * P.shape[0]))))
    g["e_pairs"] = e_pairs
    # propose_loops (fragments.cpp:61-109): 7 fragments of random clouds at scattered poses
    rng_clouds, poses = [], []
    for f in range(7):
        c = RF.random_cloud(80, 900 + f, 0, -0.4, 0.4)["source"][0]
        rng_clouds.append(c)
        Rf, tf = RF.random_transform(950 + f, 0, 0.2, 0.5)
        poses.append((Rf, tf))
    props = RF.propose_loops(rng_clouds, poses, loops=[(5, 2)], overlap_radius=0.15, min_overlap=0.1)
    g["propose_loops"] = {"clouds": [(900 + f, 80) for f in range(7)], "poses": [(950 + f, 0.2, 0.5) for f in range(7)],
                          "loops": [(5, 2)], "overlap_radius": 0.15, "min_overlap": 0.1,
                          "proposals": [(i, j, float(o).hex()) for i, j, o in props]}
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_golden.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", out)


if __name__ == "__main__":
    main()
