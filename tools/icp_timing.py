"""Config D ICP timing (diagnostic): submap pair at full resolution, ICP from
a perturbed truth; prints ms per call and per iteration."""
import sys
import time
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1801_01572_b200 as lk  # noqa: E402
from paper_1801_01572_b200 import synth  # noqa: E402

stride = int(sys.argv[1]) if len(sys.argv) > 1 else 1
t0 = time.perf_counter()
pair = synth.submap_pair(stride=stride)
print(f"fixture {pair.source.size()} / {pair.target.size()} points in {time.perf_counter() - t0:.1f} s", flush=True)
T0 = synth.compose(synth.transform_from_twist([0.02, -0.015, 0.01, 0.02, -0.01, 0.015]), pair.truth)
p = lk.IcpParams(max_correspondence_distance=0.05, max_iterations=30, convergence_eps=1e-10)
for rep in range(4):
    t0 = time.perf_counter()
    r = lk.icp_point_to_plane(pair.source, pair.target, T0, p)
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {dt * 1e3:.2f} ms, {r.iterations} iterations ({dt * 1e3 / max(len(r.history), 1):.3f} ms/it), "
          f"corr {r.correspondences}, rmse {r.rmse:.6g}, converged {r.converged}", flush=True)
