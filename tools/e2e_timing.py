"""E2E timing (diagnostic, no trace syncs): register_global on the B1 pair
from page-locked host clouds, median and min of N calls after warm-up.
usage: e2e_timing.py [reps]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_01572_b200 as lk  # noqa: E402
from paper_1801_01572_b200 import synth  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    pair = synth.depth_frame_pair()
    keep, clouds = [], []
    for c in (pair.source, pair.target):
        tp = torch.from_numpy(np.ascontiguousarray(c.positions)).pin_memory()
        tn = torch.from_numpy(np.ascontiguousarray(c.normals)).pin_memory()
        keep += [tp, tn]
        clouds.append(lk.PointCloud(tp.numpy(), tn.numpy()))
    params = lk.RegistrationParams(hypothesis_count=1_000_000, seed=1)
    for _ in range(5):
        lk.register_global(clouds[0], clouds[1], params)
    ts, idx = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = lk.register_global(clouds[0], clouds[1], params)
        ts.append(time.perf_counter() - t0)
        idx = r.hypothesis_index if r else -1
    q = sorted(ts)
    pct = {p: 1e3 * q[min(len(q) - 1, int(p / 100 * len(q)))] for p in (10, 50, 90, 99)}
    print(f"e2e median {1e3 * statistics.median(ts):.3f} ms  mean {1e3 * statistics.mean(ts):.3f} ms  "
          f"min {1e3 * min(ts):.3f} ms  p10/p50/p90/p99 {pct[10]:.3f}/{pct[50]:.3f}/{pct[90]:.3f}/{pct[99]:.3f}  "
          f"index {idx}")


if __name__ == "__main__":
    main()
