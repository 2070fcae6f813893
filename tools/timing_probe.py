"""How much of a flushed single-launch CUDA-event timing is the kernel?

For the bench's per-size FP32 pass and a few small tcgen05 network GEMMs,
times one launch between CUDA events after an L2 flush, four ways:
  flush        256 MiB write, events, launch (bench r02's method)
  clean        + a 256 MiB read after the write (the kernel starts on clean
               L2 lines instead of writing back the flush's dirty ones)
  sleep        + a device spin (torch.cuda._sleep) before the first event,
               so the host enqueue of the event + launch is hidden behind
               device work and the events bracket only device time
  clean+sleep  both
Prints one JSON line per (problem, method): median us over reps.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=9)
    args = ap.parse_args()
    import torch
    from paper_2003_06795_b200 import gemm
    dev = torch.device("cuda", 0)
    flush = torch.empty((256 << 20) // 4, device=dev)
    clean = torch.zeros((256 << 20) // 4, device=dev)
    stream = torch.cuda.current_stream()
    probs = [("f32", s, s, s) for s in (64, 128, 256, 512, 1024, 2048)]
    probs += [("bf16", 1568, 512, 2048), ("bf16", 784, 512, 4608), ("bf16", 3136, 2048, 1024),
              ("tf32", 1568, 512, 1024), ("tf32", 784, 512, 2048)]
    torch.manual_seed(0)
    for fam, m, k, n in probs:
        dt = torch.bfloat16 if fam == "bf16" else torch.float32
        a = (torch.rand(m, k, device=dev) * 2 - 1).to(dt)
        b = (torch.rand(k, n, device=dev) * 2 - 1).to(dt)
        c = torch.empty(m, n, device=dev)
        cfg = gemm.auto_config(m, k, n, family=fam)
        gemm.matmul(a, b, cfg, out=c, family=fam)
        for method in ("flush", "clean", "sleep", "clean+sleep"):
            us = []
            for _ in range(args.reps):
                flush.zero_()
                if "clean" in method:
                    clean.sum()
                if "sleep" in method:
                    torch.cuda._sleep(100_000)  # ~50 us at 1.9 GHz
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                gemm.matmul(a, b, cfg, out=c, family=fam)
                e1.record(stream)
                e1.synchronize()
                us.append(e0.elapsed_time(e1) * 1e3)
            med = statistics.median(us)
            print(json.dumps({"family": fam, "mkn": [m, k, n], "method": method,
                              "config": cfg if isinstance(cfg, str) else list(cfg.as_tuple()),
                              "us": round(med, 2),
                              "tflops": round(2.0 * m * n * k / (med * 1e-6) / 1e12, 2)}),
                  flush=True)


if __name__ == "__main__":
    main()
