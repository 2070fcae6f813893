"""VGG16 / ResNet-50 convolution layers end to end through the im2col front-end
(conv.conv2d: kp_im2col + the selector-chosen NT GEMM), per family, with
cuDNN (torch.nn.functional.conv2d, TF32 disabled for fp32) timed beside it
for context. Prints one JSON document.

    python tools/net_bench.py --batch 8 --out gpurun_out/net_bench.json
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

# (name, c_in, hw, c_out, k, stride, pad)
VGG16 = [("conv1_1", 3, 224, 64, 3, 1, 1), ("conv1_2", 64, 224, 64, 3, 1, 1),
         ("conv2_1", 64, 112, 128, 3, 1, 1), ("conv2_2", 128, 112, 128, 3, 1, 1),
         ("conv3_1", 128, 56, 256, 3, 1, 1), ("conv3_2", 256, 56, 256, 3, 1, 1),
         ("conv3_3", 256, 56, 256, 3, 1, 1), ("conv4_1", 256, 28, 512, 3, 1, 1),
         ("conv4_2", 512, 28, 512, 3, 1, 1), ("conv4_3", 512, 28, 512, 3, 1, 1),
         ("conv5_1", 512, 14, 512, 3, 1, 1), ("conv5_2", 512, 14, 512, 3, 1, 1),
         ("conv5_3", 512, 14, 512, 3, 1, 1)]
RESNET50 = [("conv1", 3, 224, 64, 7, 2, 3), ("c2_reduce", 256, 56, 64, 1, 1, 0),
            ("c2_3x3", 64, 56, 64, 3, 1, 1), ("c2_expand", 64, 56, 256, 1, 1, 0),
            ("c3_3x3", 128, 28, 128, 3, 1, 1), ("c3_expand", 128, 28, 512, 1, 1, 0),
            ("c4_3x3", 256, 14, 256, 3, 1, 1), ("c4_expand", 256, 14, 1024, 1, 1, 0),
            ("c5_3x3", 512, 7, 512, 3, 1, 1), ("c5_expand", 512, 7, 2048, 1, 1, 0)]


def time_ms(fn, reps=10):
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--families", default="f32,tf32,bf16")
    ap.add_argument("--out")
    args = ap.parse_args()
    import torch

    from paper_2003_06795_b200 import conv, gemm
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    doc = {"batch": args.batch, "networks": {}}
    for net, layers in (("vgg16", VGG16), ("resnet50", RESNET50)):
        rows = []
        for name, cin, hw, cout, k, st, pad in layers:
            g = torch.Generator(device="cpu").manual_seed(0)
            x32 = (torch.rand((args.batch, cin, hw, hw), generator=g) * 2 - 1).cuda()
            w32 = (torch.rand((cout, cin, k, k), generator=g) * 2 - 1).cuda()
            ho = (hw + 2 * pad - k) // st + 1
            flops = 2.0 * args.batch * ho * ho * cout * cin * k * k
            row = {"layer": name, "gemm_mkn": [args.batch * ho * ho, cin * k * k, cout],
                   "gflop": flops / 1e9}
            for fam in args.families.split(","):
                dt = torch.bfloat16 if fam == "bf16" else torch.float32
                x, w = x32.to(dt), w32.to(dt)
                kk = cin * k * k
                # the workspace kp_conv2d_auto needs (16-byte K pitch for the
                # tensor-core families: conv1_1 / conv1 run since round 2)
                import ctypes
                from paper_2003_06795_b200 import _native as nat
                need = ctypes.c_int64()
                d = conv._desc(x, w, st, pad)
                nat.check(nat.lib().kp_conv_workspace_elems(nat.family_id(fam), ctypes.byref(d),
                                                            ctypes.byref(need)))
                ws = torch.empty(need.value, dtype=dt, device="cuda")
                ms = time_ms(lambda: conv.conv2d(x, w, st, pad, family=fam, nhwc=True,
                                                 workspace=ws))
                im_ms = time_ms(lambda: conv.im2col(x, k, k, st, pad, family=fam))
                cfg = gemm.select(args.batch * ho * ho, kk, cout, family=fam, trans_b=True)
                row[fam] = {"ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
                            "im2col_ms": im_ms,
                            "im2col_gbs": (x.numel() + ws.numel()) * x.element_size() / im_ms / 1e6,
                            "config": list(cfg.as_tuple())}
            ref = time_ms(lambda: torch.nn.functional.conv2d(x32, w32, stride=st, padding=pad))
            row["cudnn_fp32_ms"] = ref
            rows.append(row)
            print(json.dumps(row), flush=True)
        tot = {fam: sum(r[fam]["ms"] for r in rows if "ms" in r.get(fam, {}))
               for fam in args.families.split(",")}
        doc["networks"][net] = {"layers": rows, "total_ms": tot,
                                "cudnn_fp32_total_ms": sum(r["cudnn_fp32_ms"] for r in rows)}
    print(json.dumps({k: v for k, v in doc.items() if k != "networks"} |
                     {"totals": {n: (d["total_ms"], d["cudnn_fp32_total_ms"])
                                 for n, d in doc["networks"].items()}}))
    if args.out:
        Path(args.out).write_text(json.dumps(doc, indent=1) + "\n")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
