"""Phase trace of the e2e leg of bench.py (B1): prepare_registration with
LK_TRACE=1 (host timestamps after a stream sync at every phase boundary),
then the hypotheses and the merge. Diagnostic only -- the syncs it adds make
its totals slightly larger than bench.py's e2e number."""
import os
import sys
import time

os.environ.setdefault("LK_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_01572_b200 as lk  # noqa: E402
from paper_1801_01572_b200 import synth  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    pair = synth.depth_frame_pair()
    keep, clouds = [], []
    for c in (pair.source, pair.target):
        tp = torch.from_numpy(np.ascontiguousarray(c.positions)).pin_memory()
        tn = torch.from_numpy(np.ascontiguousarray(c.normals)).pin_memory()
        keep += [tp, tn]
        clouds.append(lk.PointCloud(tp.numpy(), tn.numpy()))
    params = lk.RegistrationParams(hypothesis_count=1_000_000, seed=1)
    for r in range(reps):
        print(f"--- rep {r}", file=sys.stderr)
        t0 = time.perf_counter()
        ctx = lk.prepare_registration(clouds[0], clouds[1], params)
        t1 = time.perf_counter()
        res = lk.run_hypotheses(ctx, params)
        t2 = time.perf_counter()
        ctx.close()
        t3 = time.perf_counter()
        print(f"prepare {1e3 * (t1 - t0):.3f} ms  run+merge {1e3 * (t2 - t1):.3f} ms  close {1e3 * (t3 - t2):.3f} ms"
              f"  index {res.hypothesis_index if res else -1}", file=sys.stderr)


if __name__ == "__main__":
    main()
