"""north_star "≥ 70 % of the relevant roofline on large sizes", standalone:
bench.py's clock-sampled `large_sizes` block (every family x operand layout
at 4096^3 and 8192^3, the runtime-selected config and the best of a few
large-tile configs; FP32 against the nominal FMA-pipe peak, TF32 against
cuBLAS TF32 measured in the same process, BF16 against MEASURED_PEAKS).

    python tools/large_sizes.py > gpurun_out/large_sizes.json
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
    torch.cuda.set_device(dev)
    print(json.dumps(bench.large_sizes_block(dev, bench.family_peaks(dev))))
    return 0


if __name__ == "__main__":
    sys.exit(main())
