"""north_star "≥ 70 % of the relevant roofline on large sizes": every family x
operand layout at 4096^3 and 8192^3, the runtime-selected config and the best
of a few large-tile configs, as TFLOP/s and fraction of the roofline
(FP32: kp_fp32_peak measured in the same process; TF32/BF16: MEASURED_PEAKS
bf16 burst, TF32 = half). Warm L2 (operands far larger than L2 at 8192^3).

    python tools/large_sizes.py > gpurun_out/large_sizes.jsonl
"""
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CANDIDATES = {
    "f32": [(4, 8, 8, 32, 8), (4, 8, 8, 16, 16), (8, 8, 8, 16, 16), (2, 8, 8, 16, 16),
            (1, 8, 8, 32, 8), (4, 8, 4, 16, 16)],
    "tf32": [(4, 1, 8, 16, 16), (8, 1, 8, 16, 16), (4, 2, 8, 16, 16), (1, 1, 4, 8, 8)],
    "bf16": [(4, 1, 8, 16, 16), (8, 1, 8, 16, 16), (4, 2, 8, 16, 16), (1, 1, 4, 8, 8)],
}


def main() -> int:
    import torch
    from paper_2003_06795_b200 import _native as nat
    from paper_2003_06795_b200 import gemm
    torch.zeros(1, device="cuda")
    fp32 = ctypes.c_double()
    nat.check(nat.lib().kp_fp32_peak(ctypes.byref(fp32), None))
    bf16 = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"]) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 1590.0
    peaks = {"f32": fp32.value, "tf32": bf16 / 2, "bf16": bf16}
    for fam in ("f32", "tf32", "bf16"):
        dt = torch.bfloat16 if fam == "bf16" else torch.float32
        for s in (4096, 8192):
            for lay in ("nn", "nt", "tn", "tt"):
                g = torch.Generator(device="cpu").manual_seed(s)
                a = (torch.rand((s, s), generator=g) * 2 - 1).cuda().to(dt)
                b = (torch.rand((s, s), generator=g) * 2 - 1).cuda().to(dt)
                la = a.t() if lay[0] == "t" else a
                lb = b.t() if lay[1] == "t" else b
                sel = gemm.select(s, s, s, family=fam, trans_a=lay[0] == "t",
                                  trans_b=lay[1] == "t")
                res = {}
                for cfg in [sel.as_tuple()] + [c for c in CANDIDATES[fam] if c != sel.as_tuple()]:
                    ns = gemm.time_config(la, lb, cfg, family=fam, reps=3, warmup=2)
                    res[cfg] = 2.0 * s ** 3 / ns / 1e3
                best = max(res, key=res.get)
                print(json.dumps({
                    "family": fam, "layout": lay, "size": s, "peak_tflops": peaks[fam],
                    "selected": list(sel.as_tuple()), "selected_tflops": res[sel.as_tuple()],
                    "selected_frac": res[sel.as_tuple()] / peaks[fam],
                    "best_listed": list(best), "best_tflops": res[best],
                    "best_frac": res[best] / peaks[fam]}), flush=True)
                del a, b, la, lb
                torch.cuda.empty_cache()
    return 0


if __name__ == "__main__":
    sys.exit(main())
