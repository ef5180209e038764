import torch, time
N = 1 << 30
h = torch.empty(N, dtype=torch.uint8).pin_memory(); h.fill_(1)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
def run(nstreams, chunk):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for s in ss: s.wait_event(a)
    evs = []
    for i, off in enumerate(range(0, N, chunk)):
        s = ss[i % nstreams]
        with torch.cuda.stream(s):
            d[off:off+chunk].copy_(h[off:off+chunk], non_blocking=True)
    for s in ss:
        e = torch.cuda.Event(); e.record(s); torch.cuda.current_stream().wait_event(e)
    b.record(); torch.cuda.synchronize()
    return N / (a.elapsed_time(b) * 1e-3) / 1e9
for ns in (1, 2, 4):
    for ch in (1 << 19, 1 << 22, 1 << 25, 1 << 28):
        r = max(run(ns, ch) for _ in range(3))
        print(f"streams={ns} chunk={ch >> 10}KiB  {r:.1f} GB/s")
