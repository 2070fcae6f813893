"""A/B timing of K1 (FP32 SIMT) configs: library build x schedule mode.

    KP_LIB_PATH=paper_2003_06795_b200/libkp_prev.so python tools/k1_ab.py --tag prev
    python tools/k1_ab.py --tag new --schedules 0,1

Prints one JSON line per (size, layout, config, schedule) with the median
per-launch time (kp_gemm_time, warm L2) and TFLOP/s, and checks that every
schedule mode gives bit-identical C (ordered stream-K preserves the k order).
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

DEFAULT_CFGS = ["1,8,8,32,8", "1,8,8,16,16", "2,8,4,16,8", "2,8,8,16,16", "4,8,8,16,16",
                "4,8,4,16,16", "4,8,8,32,8", "8,8,8,16,16", "2,4,4,16,16", "4,4,8,16,16"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="new")
    ap.add_argument("--sizes", default="1024,2048,4096")
    ap.add_argument("--layouts", default="nn")
    ap.add_argument("--cfgs", default=";".join(DEFAULT_CFGS))
    ap.add_argument("--schedules", default="")
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    import torch
    from paper_2003_06795_b200 import _native as nat
    from paper_2003_06795_b200 import gemm
    scheds = [int(s) for s in args.schedules.split(",")] if args.schedules else [None]
    torch.manual_seed(0)
    for size in (int(s) for s in args.sizes.split(",")):
        m = k = n = size
        for lay in args.layouts.split(","):
            a = torch.rand((k, m) if lay[0] == "t" else (m, k), device="cuda") * 2 - 1
            b = torch.rand((n, k) if lay[1] == "t" else (k, n), device="cuda") * 2 - 1
            a = a.t() if lay[0] == "t" else a
            b = b.t() if lay[1] == "t" else b
            for cs in args.cfgs.split(";"):
                cfg = tuple(int(v) for v in cs.split(","))
                ref = None
                for sc in scheds:
                    if sc is not None:
                        nat.lib().kp_set_schedule(sc)
                    out = gemm.matmul(a, b, cfg)
                    torch.cuda.synchronize()
                    same = None
                    if ref is None:
                        ref = out.clone()
                    else:
                        same = bool(torch.equal(ref, out))
                    ns = gemm.time_config(a, b, cfg, reps=args.reps)
                    print(json.dumps({"tag": args.tag, "size": size, "layout": lay, "cfg": cfg,
                                      "schedule": sc, "us": round(ns / 1e3, 2),
                                      "tflops": round(2 * m * n * k / ns / 1e3, 2),
                                      "bit_identical": same}), flush=True)


if __name__ == "__main__":
    main()
