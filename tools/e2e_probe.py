"""e2e pipeline tuning probe: bench's square set through PinnedPipeline with
different row-block sizes (TFLOP/s end to end, pinned host buffers)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2003_06795_b200 import gemm  # noqa: E402

SIZES = (64, 128, 256, 512, 1024, 2048)
host = []
for s in SIZES:
    host.append(((torch.rand(s, s) * 2 - 1).pin_memory(), (torch.rand(s, s) * 2 - 1).pin_memory(),
                 torch.empty((s, s), pin_memory=True)))
flops = sum(2.0 * s ** 3 for s in SIZES)
for chunk_mb, graph in ((2, False), (4, False), (8, False), (2, True), (4, True), (8, True)):
    pipe = gemm.PinnedPipeline("f32", graph=graph)
    pipe.CHUNK_BYTES = chunk_mb << 20
    for _ in range(5):
        pipe.run(host)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 100
    for _ in range(n):
        pipe.run(host)
    dt = (time.perf_counter() - t0) / n
    print(json.dumps({"chunk_mb": chunk_mb, "graph": graph, "ms": round(dt * 1e3, 3), "tflops": round(flops / dt / 1e12, 2)}))
