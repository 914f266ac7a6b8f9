"""Config D pipeline (diagnostic): register_global on the 2.4M-point submap
pair (H = 10^6), then ICP on the full clouds from the global result."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1801_01572_b200 as lk  # noqa: E402
from paper_1801_01572_b200 import synth  # noqa: E402

pair = synth.submap_pair()
params = lk.RegistrationParams(hypothesis_count=1_000_000, seed=1)
for rep in range(3):
    st = lk.HypothesisStats()
    t0 = time.perf_counter()
    res = lk.register_global(pair.source, pair.target, params, st)
    t1 = time.perf_counter()
    icp = lk.icp_point_to_plane(pair.source, pair.target, res.transform, lk.IcpParams()) if res else None
    t2 = time.perf_counter()
    if res:
        R = pair.truth.rotation.T @ res.transform.rotation
        ang = np.degrees(np.arccos(np.clip((np.trace(R) - 1) / 2, -1, 1)))
        terr = np.linalg.norm(res.transform.translation - pair.truth.translation)
        R2 = pair.truth.rotation.T @ icp.transform.rotation
        ang2 = np.degrees(np.arccos(np.clip((np.trace(R2) - 1) / 2, -1, 1)))
        terr2 = np.linalg.norm(icp.transform.translation - pair.truth.translation)
        print(f"rep {rep}: register_global {1e3 * (t1 - t0):.1f} ms (evaluated {st.evaluated}, ratio "
              f"{res.inlier_ratio:.3f}; err {ang:.3f} deg {terr * 1e3:.1f} mm), ICP {1e3 * (t2 - t1):.1f} ms "
              f"({icp.iterations} it, rmse {icp.rmse:.4g}; err {ang2:.4f} deg {terr2 * 1e3:.2f} mm)", flush=True)
    else:
        print(f"rep {rep}: no alignment ({1e3 * (t1 - t0):.1f} ms)", flush=True)
