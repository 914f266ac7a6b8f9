"""Config B2 timing, diagnostic: explicit candidates on the
full-resolution depth-frame pair (no downsample) against the target's
EvalGrid; lattice around the truth at 1 deg / 1 cm."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1801_01572_b200 as lk  # noqa: E402
from paper_1801_01572_b200 import synth  # noqa: E402

half_rot = int(sys.argv[1]) if len(sys.argv) > 1 else 2
half_trans = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pair = synth.depth_frame_pair()
t0 = time.perf_counter()
grid = lk.build_eval_grid(pair.target, 0.075)
print(f"EvalGrid over {pair.target.size()} points: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
rt, ti = synth.lattice_candidates(pair.truth, math.pi / 180.0, 0.01, half_rot, half_trans)
params = lk.RegistrationParams()
for early in (True, False):
    for rep in range(2):
        t0 = time.perf_counter()
        sc = lk.score_candidates(grid, pair.source, rt, params, early_exit=early)
        dt = time.perf_counter() - t0
        evals = rt.shape[0] * pair.source.size()
        print(f"early_exit={early} C={rt.shape[0]} evals={evals:.3g} {1e3 * dt:.1f} ms "
              f"{evals / dt:.3g} evals/s best={sc.best.hypothesis_index if sc.best else None} truth={ti} "
              f"qualified={sc.qualified}", flush=True)
