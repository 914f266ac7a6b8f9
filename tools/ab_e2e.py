"""Interleaved e2e A/B of two builds of the library (diagnostic): one worker
process per .so (LK_LIB_OVERRIDE), each warmed up, then R rounds of K
register_global calls alternating between the workers, so that both see the
same box conditions (LK_AB_PAGEABLE=1: from pageable numpy clouds). Prints per-build median / min and the paired median of
per-round differences. usage: ab_e2e.py libA.so libB.so [rounds] [k]"""
import multiprocessing as mp
import os
import statistics
import sys
import time


def worker(lib, conn):
    os.environ["LK_LIB_OVERRIDE"] = os.path.abspath(lib)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    import paper_1801_01572_b200 as lk
    from paper_1801_01572_b200 import synth
    pair = synth.depth_frame_pair()
    keep, clouds = [], []
    pageable = os.environ.get("LK_AB_PAGEABLE") == "1"  # plain numpy clouds (the driver stages them)
    for c in (pair.source, pair.target):
        if pageable:
            clouds.append(lk.PointCloud(np.array(c.positions), np.array(c.normals)))
            continue
        tp = torch.from_numpy(np.ascontiguousarray(c.positions)).pin_memory()
        tn = torch.from_numpy(np.ascontiguousarray(c.normals)).pin_memory()
        keep += [tp, tn]
        clouds.append(lk.PointCloud(tp.numpy(), tn.numpy()))
    params = lk.RegistrationParams(hypothesis_count=1_000_000, seed=1)
    for _ in range(10):
        lk.register_global(clouds[0], clouds[1], params)
    conn.send("ready")
    while True:
        k = conn.recv()
        if k is None:
            return
        ts = []
        for _ in range(k):
            t0 = time.perf_counter()
            r = lk.register_global(clouds[0], clouds[1], params)
            ts.append(time.perf_counter() - t0)
        conn.send((ts, r.hypothesis_index if r else -1))


def main():
    libs = sys.argv[1:3]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    k = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    ctx = mp.get_context("spawn")
    pipes, procs = [], []
    for lib in libs:
        a, b = ctx.Pipe()
        p = ctx.Process(target=worker, args=(lib, b))
        p.start()
        pipes.append(a)
        procs.append(p)
    for a in pipes:
        assert a.recv() == "ready"
    all_t = [[], []]
    diffs = []
    for r in range(rounds):
        meds = []
        for i in (0, 1) if r % 2 == 0 else (1, 0):
            pipes[i].send(k)
            ts, idx = pipes[i].recv()
            all_t[i] += ts
            meds.append((i, statistics.median(ts)))
        m = dict(meds)
        diffs.append(m[1] - m[0])
    for a in pipes:
        a.send(None)
    for p in procs:
        p.join()
    for i, lib in enumerate(libs):
        print(f"{lib}: median {1e3 * statistics.median(all_t[i]):.3f} ms  min {1e3 * min(all_t[i]):.3f} ms")
    print(f"paired median (B - A): {1e3 * statistics.median(diffs):+.3f} ms over {rounds} rounds of {k}")


if __name__ == "__main__":
    main()
