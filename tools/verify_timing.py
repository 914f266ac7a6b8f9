"""Config E timing (diagnostic): lk_verify_batch on K synthetic pairs from
pinned host buffers, wall clock per batch; run under ncu for the launch list."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_01572_b200 as lk  # noqa: E402
from paper_1801_01572_b200 import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pairs = [synth.synth_registration_pair(s) for s in range(1, K + 1)]
keep = []


def pin(c):
    tp = torch.from_numpy(np.ascontiguousarray(c.positions)).pin_memory()
    tn = torch.from_numpy(np.ascontiguousarray(c.normals)).pin_memory()
    keep.extend([tp, tn])
    return lk.PointCloud(tp.numpy(), tn.numpy())


Q = [pin(p.target) for p in pairs]
P = [pin(p.source) for p in pairs]
I = [lk.RigidTransform() for _ in pairs]
T = [p.truth for p in pairs]
vp = lk.VerifyParams()
for r in range(reps):
    t0 = time.perf_counter()
    lk.verify_batch(Q, P, I, T, T, vp)
    print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
