"""Device timeline of one PinnedPipeline step (torch.profiler / CUPTI):
memcpy and kernel intervals relative to the step start."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2003_06795_b200 import gemm  # noqa: E402

SIZES = (64, 128, 256, 512, 1024, 2048)
host = [((torch.rand(s, s) * 2 - 1).pin_memory(), (torch.rand(s, s) * 2 - 1).pin_memory(),
         torch.empty((s, s), pin_memory=True)) for s in SIZES]
pipe = gemm.PinnedPipeline("f32")
for _ in range(5):
    pipe.run(host)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        pipe.run(host)
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
n = len(ev) // 3
step = ev[2 * n:]
t0 = step[0].time_range.start
for e in step:
    name = e.name[:60]
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f}  {e.time_range.end - e.time_range.start:7.1f}  {name}")
