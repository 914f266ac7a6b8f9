"""Multi-rank host logic on CPU (gloo, world_size 2): hypothesis sharding into
contiguous ranges, one all-reduce(sum) over a zero-filled [G x record] buffer
(an exact all-gather), and the product's exact merge -- equal to the
unsharded run. On the GPU box the same buffer is exchanged over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard_range(rank, world, H):
    return rank * H // world, (rank + 1) * H // world


def _worker(rank, world, port, H, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes as C

    import oracle as O
    import paper_1801_01572_b200 as lk
    from paper_1801_01572_b200 import abi, synth

    pair = synth.synth_registration_pair(5)
    p = O.params(hypothesis_count=H, seed=11, threads=2)
    ctx = O.Context.prepare(pair.source.positions, pair.source.normals, pair.target.positions, pair.target.normals, p)
    b, e = shard_range(rank, world, H)
    res, st = ctx.run(p, b, e)
    rec = abi.lk_reg_record()
    rec.valid = int(res.found)
    rec.inliers = res.inliers
    rec.fitness = res.fitness
    rec.index = res.hypothesis_index
    for k in range(9):
        rec.R[k] = res.R.reshape(9)[k]
    for k in range(3):
        rec.t[k] = res.t[k]
    for k in ("sampled", "prerejected", "degenerate", "evaluated", "qualified", "w_ref"):
        setattr(rec, k, st[k])
    words = C.sizeof(abi.lk_reg_record) // 8
    buf = torch.zeros(world * words, dtype=torch.int64)
    buf[rank * words:(rank + 1) * words] = torch.from_numpy(np.frombuffer(bytes(rec), dtype=np.int64).copy())
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    recs = lk.records_from_bytes(buf.numpy())
    merged_stats = lk.HypothesisStats()
    merged = lk.merge_records(recs, ctx.ns, merged_stats)
    if rank == 0:
        full, fst = ctx.run(p)
        out_q.put(dict(
            idx=(merged.hypothesis_index, full.hypothesis_index),
            inl=(merged.inliers, full.inliers),
            fit=(merged.fitness, full.fitness),
            R=(merged.transform.rotation.tobytes(), full.R.tobytes()),
            stats=({k: getattr(merged_stats, k) for k in ("sampled", "prerejected", "degenerate", "evaluated",
                                                           "qualified", "w_ref")},
                   {k: fst[k] for k in ("sampled", "prerejected", "degenerate", "evaluated", "qualified", "w_ref")})))
    dist.destroy_process_group()


def test_shard_ranges_cover_exactly():
    for H in (0, 1, 7, 1_000_000, 4_000_003):
        for world in (1, 2, 4, 8):
            rs = [shard_range(g, world, H) for g in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == H
            assert all(rs[g][1] == rs[g + 1][0] for g in range(world - 1))


@pytest.mark.timeout(300)
def test_two_rank_exchange_equals_single_run():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 20_000, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=280)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for k in ("idx", "inl", "fit", "R", "stats"):
        assert out[k][0] == out[k][1], k
