"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep --key f32_nn_4096_1-8-8-16-16 \
        --flops 1.37e11 --out profiles/ncu_r01.md

Appends a markdown section (duration, SM/DRAM throughput, FMA / tensor pipe
utilisation, issue-slot use, registers, occupancy, dram bytes, top stall
reasons, instruction mix) and records dram bytes per launch in
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

METRICS = {
    "gpu__time_duration.sum": "duration",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_cycles_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def ncu_csv(rep: Path, page: str, extra=()):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", page, "--csv", *extra],
                         capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep: Path) -> dict:
    rows = ncu_csv(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    got = {}
    for key, name in METRICS.items():
        if key in hdr:
            i = hdr.index(key)
            got[name] = (vals[i], units[i])
    stalls = {}
    for i, k in enumerate(hdr):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i])
            except ValueError:
                pass
    name_i = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
    return {"metrics": got, "stalls": stalls, "kernel": vals[name_i] if name_i is not None else ""}


def instruction_mix(rep: Path, top: int = 10):
    rows = ncu_csv(rep, "source", ["--print-source", "sass"])
    hdr = rows[1]
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    mix, total = collections.Counter(), 0
    for r in rows[2:]:
        try:
            n = int(r[i_ex])
        except (ValueError, IndexError):
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        mix[op] += n
        total += n
    return [(op, n, 100.0 * n / total) for op, n in mix.most_common(top)], total


def to_float(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--key", required=True)
    ap.add_argument("--flops", type=float, help="algorithmic flops of the launch")
    ap.add_argument("--bytes", type=float, help="algorithmic bytes of the launch")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "ncu_summary.md"))
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    rep = Path(args.rep)
    raw = raw_metrics(rep)
    m = raw["metrics"]
    lines = [f"\n## {args.key}\n", f"`{raw['kernel'][:160]}`  \n", f"capture: `{rep.name}` "
             f"(ncu --set full --clock-control none)  \n"]
    if args.note:
        lines.append(args.note + "  \n")
    lines.append("\n| metric | value |\n|---|---|\n")
    for name, (val, unit) in m.items():
        lines.append(f"| {name} | {val} {unit} |\n")
    dur = m.get("duration")
    if dur and args.flops:
        d = to_float(dur[0])
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
                 "nsecond": 1e-9}.get(dur[1], 1e-9)
        if d:
            lines.append(f"| achieved (cold, serialised) | {args.flops / (d * scale) / 1e12:.2f} "
                         f"TFLOP/s |\n")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    dram_bytes = sum((to_float(m.get(k, ("0", "byte"))[0]) or 0) *
                     scale.get(m.get(k, ("0", "byte"))[1], 1) for k in ("dram_read", "dram_write"))
    lines.append(f"| dram traffic | {dram_bytes / 1e6:.2f} MB"
                 + (f" (algorithmic {args.bytes / 1e6:.2f} MB)" if args.bytes else "") + " |\n")
    st = sorted(raw["stalls"].items(), key=lambda kv: -kv[1])[:6]
    tot = sum(raw["stalls"].values()) or 1
    lines.append("\nTop stall reasons (pc samples): "
                 + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in st) + "\n")
    try:
        mix, total = instruction_mix(rep)
        lines.append("\nInstruction mix: " + ", ".join(f"{op} {pct:.1f}%" for op, _, pct in mix)
                     + f" (total {total:.3g} warp-instructions)\n")
    except Exception as exc:  # noqa: BLE001
        lines.append(f"\n(instruction mix unavailable: {exc})\n")
    out = Path(args.out)
    out.parent.mkdir(exist_ok=True)
    with open(out, "a") as fh:
        fh.writelines(lines)
    tpath = ROOT / "profiles" / "ncu_traffic.json"
    doc = json.loads(tpath.read_text()) if tpath.exists() else {}
    doc[args.key] = {"dram_bytes": dram_bytes, "capture": rep.name}
    tpath.write_text(json.dumps(doc, indent=1) + "\n")
    print("".join(lines))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
