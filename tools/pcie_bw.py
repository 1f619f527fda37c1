import torch, time
n = 2 * 1024**3  # 2 GiB
d = torch.empty(n, dtype=torch.uint8, device='cuda')
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for name, f in [('d2h', lambda: h.copy_(d, non_blocking=True)), ('h2d', lambda: d.copy_(h, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    best = 0
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    print(name, 'GB/s', round(best, 1))
# bidirectional: both at once on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty(n, dtype=torch.uint8, device='cuda'); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize(); t = time.time()
with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize(); print('bidir GB/s each', round(n / (time.time() - t) / 1e9, 1))
