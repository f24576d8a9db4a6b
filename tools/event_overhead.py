import torch
x = torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    x.add_(1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        x.add_(1)
        x.add_(1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for mode in ("graph2", "direct2"):
        ts = []
        for i in range(30):
            flush.fill_(i & 0xff)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if mode == "graph2": g.replay()
            else: x.add_(1); x.add_(1)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(mode, "event pair us: median", round(ts[15], 2), "min", round(ts[0], 2))
