"""Check: can timing events be captured inside a CUDA graph and read after replay?"""
import torch
x = torch.randn(1 << 24, device="cuda")
y = torch.empty_like(x)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        y.copy_(x)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
try:
    with torch.cuda.graph(g):
        e0.record()
        for _ in range(10):
            y.copy_(x)
        e1.record()
    g.replay()
    torch.cuda.synchronize()
    print("in-graph events ok:", e0.elapsed_time(e1), "ms for 10 copies of 64 MB")
except Exception as exc:
    print("in-graph events FAILED:", repr(exc))
