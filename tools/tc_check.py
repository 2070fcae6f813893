"""Correctness probe for the tcgen05 families (prints errors instead of asserting)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2003_06795_b200 import gemm


def check(fam, cfg, m, k, n, trans):
    dt = torch.bfloat16 if fam == "bf16" else torch.float32
    g = torch.Generator().manual_seed(0)
    a = (torch.rand((k, m) if trans[0] == "t" else (m, k), generator=g) * 2 - 1).to(dt).cuda()
    b = (torch.rand((n, k) if trans[1] == "t" else (k, n), generator=g) * 2 - 1).to(dt).cuda()
    a = a.t() if trans[0] == "t" else a
    b = b.t() if trans[1] == "t" else b
    try:
        c = gemm.matmul(a, b, cfg, family=fam)
        torch.cuda.synchronize()
    except Exception as exc:
        print(f"{fam} {trans} {cfg} {(m, k, n)}: ERROR {exc}")
        return False
    ref = a.double().cpu() @ b.double().cpu()
    err = (c.double().cpu() - ref).abs().max().item()
    rel = ((c.double().cpu() - ref).norm() / ref.norm()).item()
    print(f"{fam} {trans} {cfg} {(m, k, n)}: max_abs {err:.3e} rel {rel:.3e}")
    return rel < 1e-2


if __name__ == "__main__":
    fams = sys.argv[1].split(",") if len(sys.argv) > 1 else ["tf32", "bf16"]
    for fam in fams:
        for trans in ("tn", "nn", "nt", "tt"):
            for cfg in [(1, 1, 1, 8, 8), (4, 1, 8, 16, 16), (4, 2, 4, 16, 16), (4, 2, 8, 16, 16)]:
                check(fam, cfg, 520, 264, 776, trans)
