"""Pinned host<->device copy bandwidth on this box (the e2e ceiling)."""
import json
import torch

x = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty_like(x, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name in ("h2d", "d2h", "both"):
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        if name in ("h2d", "both"):
            with torch.cuda.stream(s_in):
                d.copy_(x, non_blocking=True)
        if name in ("d2h", "both"):
            y = torch.empty_like(x).pin_memory() if name == "both" else x
            with torch.cuda.stream(s_out):
                y.copy_(d if name == "d2h" else torch.empty_like(d), non_blocking=True)
        torch.cuda.current_stream().wait_stream(s_in)
        torch.cuda.current_stream().wait_stream(s_out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    res[name + "_GBps"] = round((x.numel() * (2 if name == "both" else 1)) / ms / 1e6, 1)
print(json.dumps(res))
