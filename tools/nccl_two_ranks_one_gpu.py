import multiprocessing as mp, sys
sys.path.insert(0, '.')
def main(rank, uid, q):
    try:
        import paper_1801_01572_b200 as lk
        from paper_1801_01572_b200 import synth
        pr = synth.synth_registration_pair(1)
        p = lk.RegistrationParams(hypothesis_count=40000, seed=5, device=0)
        ctx = lk.prepare_registration(pr.source, pr.target, p)
        ctx.attach_comm(uid, 2, rank)
        st = lk.HypothesisStats(); r = lk.run_hypotheses(ctx, p, st)
        q.put((rank, r.hypothesis_index, st.w_ref))
    except Exception as e:
        q.put((rank, 'error', repr(e)))
if __name__ == '__main__':
    import paper_1801_01572_b200 as lk
    uid = lk.nccl_unique_id()
    c = mp.get_context('spawn'); q = c.Queue()
    ps = [c.Process(target=main, args=(r, uid, q)) for r in range(2)]
    [p.start() for p in ps]
    print([q.get(timeout=300) for _ in ps]); [p.join(60) for p in ps]
