"""FC-layer (m <= 16) throughput of the small-M path vs the selected tile
config: bench.small_m_block standalone, one JSON line per family.

    python tools/skinny_probe.py > gpurun_out/skinny_probe.jsonl
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> int:
    import torch
    import bench
    dev = torch.device("cuda", 0)
    torch.zeros(1, device=dev)
    peaks = {"_hbm_gbs": bench.measured_peaks()["hbm_gbs"]}
    out = bench.small_m_block(dev, peaks)
    for fam, blk in out.items():
        print(json.dumps({"family": fam, **{k: v for k, v in blk.items() if k != "rows"}}))
        for r in blk["rows"]:
            print(json.dumps({"family": fam, **r}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
