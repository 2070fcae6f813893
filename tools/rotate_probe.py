"""Single flushed launch vs back-to-back launches over rotated operand sets.

For the network_roofline problems of one family (bench.py's set: configs[2],
>= 1 GFLOP, AI >= ridge), times kp_gemm_auto's pick two ways:
  flushed   one launch between CUDA events after a 256 MiB L2 flush (bench
            r02's network_roofline method; the events also hold the
            launch latency of that one kernel)
  rotated   R back-to-back launches between one pair of events, cycling over
            enough distinct (A, B, C) sets that their total exceeds 160 MB
            (> the 126 MB L2), so no launch finds its operands in L2; the
            per-launch figure is the window / R
One JSON line per problem.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--family", default="bf16")
    ap.add_argument("--launches", type=int, default=60)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2003_06795_b200 import gemm
    from paper_2003_06795_b200.shapes import network_problems
    dev = torch.device("cuda", 0)
    peaks = bench.family_peaks(dev)
    fam = args.family
    peak = peaks[fam][0]
    es = 2 if fam == "bf16" else 4
    ridge = peak * 1e12 / (peaks["_hbm_gbs"] * 1e9)
    probs = [p for p in network_problems()
             if 2.0 * p.m * p.n * p.k >= 1e9
             and 2.0 * p.m * p.n * p.k / (es * (p.m * p.k + p.k * p.n) + 4 * p.m * p.n) >= ridge]
    flush = torch.empty((256 << 20) // 4, device=dev)
    stream = torch.cuda.current_stream()
    for i, p in enumerate(probs):
        set_bytes = es * (p.m * p.k + p.k * p.n) + 4 * p.m * p.n
        nsets = max(2, -(-(160 << 20) // set_bytes))
        if nsets * set_bytes > (8 << 30):
            continue
        sets = []
        for s in range(nsets):
            a, b = bench.device_operands(p.m, p.k, p.n, fam, False, False, dev, 500 + s)
            sets.append((a, b, torch.empty((p.m, p.n), device=dev)))
        cfg = gemm.auto_config(p.m, p.k, p.n, family=fam)
        for a, b, c in sets:
            gemm.matmul(a, b, cfg, out=c, family=fam)
        single = []
        for _ in range(5):
            a, b, c = sets[0]
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gemm.matmul(a, b, cfg, out=c, family=fam)
            e1.record(stream)
            e1.synchronize()
            single.append(e0.elapsed_time(e1) * 1e3)
        rot = []
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for j in range(args.launches):
                a, b, c = sets[j % nsets]
                gemm.matmul(a, b, cfg, out=c, family=fam)
            e1.record(stream)
            e1.synchronize()
            rot.append(e0.elapsed_time(e1) * 1e3 / args.launches)
        fl = 2.0 * p.m * p.n * p.k
        t1, t2 = statistics.median(single), statistics.median(rot)
        print(json.dumps({"family": fam, "mkn": [p.m, p.k, p.n],
                          "config": cfg if isinstance(cfg, str) else list(cfg.as_tuple()),
                          "sets": nsets, "flushed_us": round(t1, 2), "rotated_us": round(t2, 2),
                          "flushed_frac": round(fl / (t1 * 1e-6) / 1e12 / peak, 4),
                          "rotated_frac": round(fl / (t2 * 1e-6) / 1e12 / peak, 4)}), flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
