"""Phase timeline of the tcgen05 1-CTA kernel from a KP_TC_DEBUG build.

    python -m paper_2003_06795_b200.build --debug      (libkp_debug.so)
    KP_LIB_PATH=paper_2003_06795_b200/libkp_debug.so \\
        python tools/tc_trace.py --family bf16 --mkn 1024,1024,1024 --cfg 1,1,4,8,8

Per-CTA %globaltimer stamps (0 entry, 1 setup done, 2 first TMA issued,
3 first stage landed, 4 last MMA issued, 5 accumulator complete, 6 stores
issued, 7 exit); prints the median / max of each phase relative to the
earliest CTA entry, one JSON line.
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

NAMES = ("entry", "setup", "first_tma", "first_landed", "last_mma", "acc_full", "stored", "exit",
         "epi_c0_regs", "epi_c0_issued", "epi_c1_regs", "epi_c1_issued", "epi_c2_regs",
         "epi_c2_issued", "epi_c3_regs", "epi_c3_issued")


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--family", default="bf16")
    ap.add_argument("--mkn", default="1024,1024,1024")
    ap.add_argument("--cfg", default="1,1,4,8,8")
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2003_06795_b200 import _native as nat, gemm
    m, k, n = (int(v) for v in args.mkn.split(","))
    cfg = tuple(int(v) for v in args.cfg.split(","))
    dt = torch.bfloat16 if args.family == "bf16" else torch.float32
    a = torch.rand(m, k, device="cuda").to(dt)
    b = torch.rand(k, n, device="cuda").to(dt)
    for _ in range(args.iters):
        gemm.matmul(a, b, cfg, family=args.family)
    torch.cuda.synchronize()
    lib = nat.lib()
    ctas = min(4096, 148 if cfg[3] == 16 else -(-m // 128) * -(-n // (32 * cfg[2])))
    buf = (ctypes.c_ulonglong * (ctas * 16))()
    if lib.kp_tc_trace_dump(buf, ctas) != 0:
        print("kp_tc_trace_dump failed (not a KP_TC_DEBUG build?)", file=sys.stderr)
        return 1
    t = np.array(buf, dtype=np.float64).reshape(ctas, 16)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3  # us
    out = {"family": args.family, "mkn": [m, k, n], "cfg": list(cfg), "ctas": ctas,
           "median_us": {nm: round(float(np.median(rel[:, i])), 3) for i, nm in enumerate(NAMES)},
           "max_us": {nm: round(float(rel[:, i].max()), 3) for i, nm in enumerate(NAMES)},
           "phase_median_us": {f"{NAMES[i]}->{NAMES[i + 1]}":
                               round(float(np.median(rel[:, i + 1] - rel[:, i])), 3)
                               for i in range(15)}}
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
