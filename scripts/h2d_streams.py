import torch, time
n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]
def run(k, chunk=16 << 20, reps=10):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in ss[:k]: s.wait_event(e0)
        for i, off in enumerate(range(0, n, chunk)):
            s = ss[i % k]
            with torch.cuda.stream(s):
                d[off:off+chunk].copy_(h[off:off+chunk], non_blocking=True)
        for s in ss[:k]:
            ev = torch.cuda.Event(); ev.record(s); torch.cuda.current_stream().wait_event(ev)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return n / best / 1e6
for k in (1, 2, 4):
    for c in (4 << 20, 16 << 20, 64 << 20):
        print(k, c >> 20, "MiB", round(run(k, c), 2), "GB/s")
