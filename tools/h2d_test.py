import torch, time
N = 307200*3
a = [torch.randn(N, dtype=torch.float64).pin_memory() for _ in range(4)]
d = [torch.empty(N, dtype=torch.float64, device='cuda') for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
    e0.record(s1); s2.wait_event(e0)
    with torch.cuda.stream(s1):
        d[0].copy_(a[0], non_blocking=True); d[1].copy_(a[1], non_blocking=True)
        e1.record(s1)
    with torch.cuda.stream(s2):
        d[2].copy_(a[2], non_blocking=True); d[3].copy_(a[3], non_blocking=True)
        e2.record(s2)
    torch.cuda.synchronize()
    print("two streams: s1 done %.3f ms, s2 done %.3f ms" % (e0.elapsed_time(e1), e0.elapsed_time(e2)))
    torch.cuda.synchronize()
    e0.record(s1)
    with torch.cuda.stream(s1):
        for k in range(4): d[k].copy_(a[k], non_blocking=True)
        e1.record(s1)
    torch.cuda.synchronize()
    print("one stream 4 copies: %.3f ms (%.1f GB/s)" % (e0.elapsed_time(e1), 4*N*8/e0.elapsed_time(e1)/1e6))
