"""Multi-GPU inside the library (include/loopkit_b200.h: lk_reg_params.device_count,
lk_nccl_unique_id / lk_reg_ctx_attach_comm / lk_reg_run_exchange, lk_verify_params.device_count).

SURVEY.md 8e: hypothesis i is a pure function of (seed, i) and selection is a
strict total order, so any sharding gives the 1-GPU result bit for bit. These
run on however many B200s the box has: with one GPU the G > 1 cases check the
error path, and the NCCL code runs with one rank (ncclCommInitRank +
ncclAllReduce over a 1-rank communicator)."""
import json
import multiprocessing as mp
import os

import numpy as np
import pytest

import paper_1801_01572_b200 as lk
from paper_1801_01572_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if lk.device_count() == 0:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")


@pytest.fixture(scope="module")
def pair():
    return synth.synth_registration_pair(1)


def _same(a, b, sa, sb):
    assert (a is None) == (b is None)
    if a is not None:
        assert a.hypothesis_index == b.hypothesis_index and a.inliers == b.inliers
        assert a.fitness == b.fitness and np.array_equal(a.transform.rotation, b.transform.rotation)
        assert np.array_equal(a.transform.translation, b.transform.translation)
    for k in ("sampled", "prerejected", "degenerate", "evaluated", "qualified", "w_ref"):
        assert getattr(sa, k) == getattr(sb, k), k


def test_device_count_all_visible_equals_one(pair):
    p1 = lk.RegistrationParams(hypothesis_count=50_000, seed=3)
    s1 = lk.HypothesisStats()
    r1 = lk.register_global(pair.source, pair.target, p1, s1)
    pg = lk.RegistrationParams(hypothesis_count=50_000, seed=3, device=0, device_count=-1)
    sg = lk.HypothesisStats()
    rg = lk.register_global(pair.source, pair.target, pg, sg)
    _same(r1, rg, s1, sg)
    ctx = lk.prepare_registration(pair.source, pair.target, pg)
    assert ctx.topology()[0] == lk.device_count()


def test_device_count_two(pair):
    p = lk.RegistrationParams(hypothesis_count=50_000, seed=3, device=0, device_count=2)
    if lk.device_count() < 2:
        with pytest.raises(lk.Error):
            lk.register_global(pair.source, pair.target, p)
        return
    s1, s2 = lk.HypothesisStats(), lk.HypothesisStats()
    r1 = lk.register_global(pair.source, pair.target, lk.RegistrationParams(hypothesis_count=50_000, seed=3), s1)
    r2 = lk.register_global(pair.source, pair.target, p, s2)
    _same(r1, r2, s1, s2)


def test_attach_comm_single_rank_equals_plain_run(pair):
    """ncclCommInitRank + the NCCL record exchange with one rank."""
    p = lk.RegistrationParams(hypothesis_count=40_000, seed=5)
    ctx = lk.prepare_registration(pair.source, pair.target, p)
    s1 = lk.HypothesisStats()
    r1 = lk.run_hypotheses(ctx, p, s1)
    ctx.attach_comm(lk.nccl_unique_id(), 1, 0)
    assert ctx.topology() == (1, 1, 0)
    s2 = lk.HypothesisStats()
    r2 = lk.run_hypotheses(ctx, p, s2)
    _same(r1, r2, s1, s2)
    with pytest.raises(lk.Error):
        ctx.attach_comm(lk.nccl_unique_id(), 1, 0)  # one communicator per context


def _rank_main(rank, nranks, uid, q):
    try:
        import paper_1801_01572_b200 as lk2
        from paper_1801_01572_b200 import synth as sy
        pr = sy.synth_registration_pair(1)
        p = lk2.RegistrationParams(hypothesis_count=40_000, seed=5, device=rank % lk2.device_count())
        ctx = lk2.prepare_registration(pr.source, pr.target, p)
        ctx.attach_comm(uid, nranks, rank)
        st = lk2.HypothesisStats()
        r = lk2.run_hypotheses(ctx, p, st)
        q.put((rank, r.hypothesis_index if r else -1, r.fitness if r else 0.0, st.w_ref, st.evaluated))
    except Exception as e:  # reported to the parent
        q.put((rank, "error", repr(e)))


def test_two_ranks_one_process_each(pair):
    """Two processes, one rank each, exchanging over NCCL: every rank returns
    the 1-GPU result. Needs two GPUs (NCCL refuses two ranks on one device)."""
    if lk.device_count() < 2:
        pytest.skip("one GPU: NCCL does not put two ranks on one device")
    ctx_m = mp.get_context("spawn")
    q = ctx_m.Queue()
    uid = lk.nccl_unique_id()
    procs = [ctx_m.Process(target=_rank_main, args=(r, 2, uid, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=600) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(o[1] != "error" for o in out), out
    p = lk.RegistrationParams(hypothesis_count=40_000, seed=5)
    st = lk.HypothesisStats()
    r = lk.register_global(pair.source, pair.target, p, st)
    for o in out:
        assert o[1] == r.hypothesis_index and o[2] == r.fitness and o[3] == st.w_ref and o[4] == st.evaluated


def test_verify_batch_device_count(pair):
    pairs = [synth.synth_registration_pair(s) for s in (1, 3)]
    Q = [p.target for p in pairs]
    P = [p.source for p in pairs]
    I = [lk.RigidTransform() for _ in pairs]
    T = [p.truth for p in pairs]
    base = lk.verify_batch(Q, P, I, T, T, lk.VerifyParams())
    allv = lk.verify_batch(Q, P, I, T, T, lk.VerifyParams(device=0, device_count=-1))
    for a, b in zip(base, allv):
        assert a.info.pair_count == b.info.pair_count and np.array_equal(a.info.info, b.info.info)
        assert a.overlap_hits == b.overlap_hits and a.inliers == b.inliers and a.fitness == b.fitness
    if lk.device_count() < 2:
        with pytest.raises(lk.Error):
            lk.verify_batch(Q, P, I, T, T, lk.VerifyParams(device=0, device_count=2))


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_multi_rank_product_path_one_device():
    """bench.py's N > 1 path -- contiguous hypothesis shares per rank, the rank
    records exchanged and merged -- with two ranks on cuda:0 (LK_BENCH_ONE_DEVICE:
    gloo carries the exchange, since NCCL refuses two ranks on one device). The
    merged result must be the reference's B1 result (tests/golden/ref_golden.json)."""
    import json as _json
    import subprocess
    import sys
    g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden.json")))["b1"]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LK_BENCH_ONE_DEVICE="1", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--e2e-steps", "2", "--no-extras", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = _json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["hypothesis_index"] == g["index"]
    assert {k: line["stats_per_step"][k] for k in g["stats"]} == g["stats"]
    assert line["stats_per_step"]["w_ref"] == g["oracle_w_ref"]


def test_concurrent_register_global_from_threads():
    """Host threads calling lk_register_global at once (ctypes releases the
    GIL): each call owns its context, streams, worker and pinned staging, so
    every result equals the same call made alone."""
    import threading
    pairs = [synth.synth_registration_pair(s) for s in (1, 2, 3, 4)]
    p = lk.RegistrationParams(hypothesis_count=60_000, seed=7)
    alone = []
    for pr in pairs:
        st = lk.HypothesisStats()
        alone.append((lk.register_global(pr.source, pr.target, p, st), st))
    got = [None] * len(pairs)
    errs = []

    def work(k):
        try:
            for _ in range(3):
                st = lk.HypothesisStats()
                got[k] = (lk.register_global(pairs[k].source, pairs[k].target, p, st), st)
        except Exception as e:  # reported below
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(pairs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (ra, sa), (rb, sb) in zip(alone, got):
        _same(ra, rb, sa, sb)
