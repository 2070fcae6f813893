"""Pinned host<->device copy bandwidth on this box (the e2e ceiling):
one direction at a time, then both directions concurrently."""
import json
import torch

n = 64 << 20
hx, hy = torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.uint8).pin_memory()
dx, dy = torch.empty(n, dtype=torch.uint8, device="cuda"), torch.empty(n, dtype=torch.uint8, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name in ("h2d", "d2h", "both"):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s_in.wait_stream(torch.cuda.current_stream())
        s_out.wait_stream(torch.cuda.current_stream())
        if name in ("h2d", "both"):
            with torch.cuda.stream(s_in):
                dx.copy_(hx, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s_out):
                hy.copy_(dy, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s_in)
        torch.cuda.current_stream().wait_stream(s_out)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[name + "_GBps"] = round(n * (2 if name == "both" else 1) / best / 1e6, 1)
print(json.dumps(res))
