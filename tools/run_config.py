"""Launch one config on one problem a few times (for ncu captures).

    python tools/run_config.py --mkn 2048,2048,2048 --cfg 4,8,8,16,16 --iters 3
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mkn", default="2048,2048,2048")
    ap.add_argument("--cfg", default="4,8,8,16,16")
    ap.add_argument("--family", default="f32")
    ap.add_argument("--trans", default="nn")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--schedule", type=int, help="K1 tile schedule (kp_set_schedule)")
    ap.add_argument("--tc-split", type=int, help="tcgen05 split-K mode (kp_set_tc_split)")
    ap.add_argument("--no-time", action="store_true", help="launch only (sanitizer runs)")
    args = ap.parse_args()
    import torch
    from paper_2003_06795_b200 import gemm
    m, k, n = (int(v) for v in args.mkn.split(","))
    cfg = tuple(int(v) for v in args.cfg.split(","))
    dt = torch.bfloat16 if args.family == "bf16" else torch.float32
    a = torch.rand((k, m) if args.trans[0] == "t" else (m, k), device="cuda").to(dt)
    b = torch.rand((n, k) if args.trans[1] == "t" else (k, n), device="cuda").to(dt)
    a = a.t() if args.trans[0] == "t" else a
    b = b.t() if args.trans[1] == "t" else b
    if args.schedule is not None:
        from paper_2003_06795_b200 import _native as nat
        nat.lib().kp_set_schedule(args.schedule)
    if args.tc_split is not None:
        from paper_2003_06795_b200 import _native as nat
        nat.lib().kp_set_tc_split(args.tc_split)
    for _ in range(args.iters):
        gemm.matmul(a, b, cfg, family=args.family)
    torch.cuda.synchronize()
    if args.no_time:
        print(f"{args.family} {args.trans} {(m, k, n)} cfg={cfg}: launched {args.iters}x")
        return
    ns = gemm.time_config(a, b, cfg, family=args.family, reps=5)
    print(f"{args.family} {args.trans} {(m, k, n)} cfg={cfg}: {ns/1e3:.1f} us, "
          f"{2*m*n*k/ns/1e3:.2f} TFLOP/s")


if __name__ == "__main__":
    main()
