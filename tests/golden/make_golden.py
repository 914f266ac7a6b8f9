"""Generates tests/golden/golden.json from the CPU oracle (itself pinned by the
reference's known-answer tests, tests/test_oracle_*.py). The reference ships
no golden files and cannot be built here (Eigen absent), so these vectors
freeze the oracle's outputs: tests check the oracle and the B200 path against
them. Re-run only when the oracle's restatement deliberately changes.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_1801_01572_b200 import synth  # noqa: E402


def hexd(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).reshape(-1)]


def main():
    g = {"about": __doc__.strip().splitlines()[0]}
    g["rng_u64"] = {f"{s},{k}": [int(x) for x in O.rng_u64(s, k, 8)] for s, k in [(0, 0), (1, 0), (99, 5)]}
    g["rng_bounded"] = {f"{s},{k},{b}": [int(x) for x in O.rng_bounded(s, k, b, 16)]
                        for s, k, b in [(7, 3, 10), (1, 2, 5309), (3, 4, 2**31 + 11)]}
    rng = np.random.default_rng(2024)
    kab = []
    for _ in range(8):
        s = rng.normal(size=(4, 3))
        T = synth.random_transform(int(rng.integers(1 << 30)), 0)
        d = s @ T.rotation.T + T.translation + 0.01 * rng.normal(size=(4, 3))
        R, t = O.kabsch(s, d)
        kab.append({"src": hexd(s), "dst": hexd(d), "R": hexd(R), "t": hexd(t)})
    g["kabsch"] = kab
    runs = []
    for seed_pair in (1, 2):
        pair = synth.synth_registration_pair(seed_pair)
        fx = {"pair": seed_pair, "n_src": pair.source.size(), "n_tgt": pair.target.size(),
              "src_sum": float(pair.source.positions.sum()).hex(), "tgt_sum": float(pair.target.positions.sum()).hex()}
        for seed, H in ((1, 20_000), (7, 20_000)):
            p = O.params(hypothesis_count=H, seed=seed)
            ctx = O.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions,
                                    pair.target.normals, p)
            r, st = ctx.run(p)
            c = ctx.get()
            runs.append(dict(fx, seed=seed, H=H, ns=ctx.ns, nt=ctx.nt,
                             cache_sum=int(c["cache"].astype(np.int64).sum()),
                             found=r.found, index=r.hypothesis_index, inliers=r.inliers,
                             fitness=float(r.fitness).hex(), R=hexd(r.R), t=hexd(r.t),
                             stats={k: st[k] for k in ("sampled", "prerejected", "degenerate", "evaluated",
                                                       "qualified", "w_ref")}))
    g["run_hypotheses"] = runs
    pair = synth.surface_pair(1, density=150.0)
    rt, truth_idx = synth.lattice_candidates(pair.truth, half_rot=1, half_trans=1)
    ref = O.score_candidates(pair.source.positions, pair.source.normals, pair.target.positions,
                             pair.target.normals, rt, 1, 0, 0.075, O.params())
    g["score_candidates"] = {"seed": 1, "density": 150.0, "half_rot": 1, "half_trans": 1, "truth_index": truth_idx,
                             "inliers": [int(x) for x in ref["inliers"]], "fitness": hexd(ref["fitness"]),
                             "best": ref["best"].hypothesis_index, "qualified": ref["qualified"]}
    pair = synth.synth_registration_pair(1)
    info, cnt = O.edge_info(pair.target.positions, pair.source.positions, np.eye(3), np.zeros(3),
                            pair.truth.rotation, pair.truth.translation, 0.05)
    g["edge_info"] = {"pair": 1, "eps": 0.05, "pair_count": cnt, "info": [float(x) for x in info.reshape(-1)]}
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
