"""In-tree build of libkp.so (sm_100a) and of the CPU oracle library.

nvcc cross-compiles for `-gencode arch=compute_100a,code=sm_100a` without a
GPU, so this runs in the CPU container as well as on the B200 box. Objects go
to ``paper_2003_06795_b200/_build`` and are rebuilt only when a source or
header is newer; the 16 K1 instantiation units compile in parallel.

    python -m paper_2003_06795_b200.build            # library + oracle
    python -m paper_2003_06795_b200.build --force
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libkp.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "liboracle_gemm.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
TILES = (1, 2, 4, 8)


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _units():
    """(object name, source, extra defines) for every translation unit."""
    units = [("kp_abi.o", CSRC / "kp_abi.cu", []),
             ("tc_gemm.o", CSRC / "tc_gemm.cu", []),
             ("peak.o", CSRC / "peak.cu", [])]
    for acc in TILES:
        for rt in TILES:
            units.append((f"simt_a{acc}_r{rt}.o", CSRC / "simt_inst.cu",
                          [f"-DKP_ACC={acc}", f"-DKP_RT={rt}"]))
    return units


def _newest_header() -> float:
    paths = list(CSRC.rglob("*.cuh")) + list(CSRC.rglob("*.h")) + [ROOT / "include" / "kp_abi.h"]
    return max(p.stat().st_mtime for p in paths if p.exists())


def _compile(name, src, defines, force, verbose):
    out = OBJ / name
    if not force and out.exists():
        stamp = out.stat().st_mtime
        if stamp >= src.stat().st_mtime and stamp >= _newest_header():
            return name, False
    cmd = [nvcc()] + NVCC_FLAGS + defines + ["-c", str(src), "-o", str(out)]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{res.stderr}")
    return name, True


def build_library(force: bool = False, verbose: bool = False, jobs: int | None = None,
                  debug: bool = False) -> Path:
    """Build libkp.so (debug=True: libkp_debug.so with -DKP_TC_DEBUG watchdog prints)."""
    global OBJ, LIB
    if debug:
        OBJ, LIB = PKG / "_build_debug", PKG / "libkp_debug.so"
    OBJ.mkdir(exist_ok=True)
    units = [(n, s, d + (["-DKP_TC_DEBUG"] if debug else [])) for n, s, d in _units()]
    jobs = jobs or max(1, os.cpu_count() or 1)
    changed = False
    with cf.ThreadPoolExecutor(max_workers=jobs) as pool:
        futs = [pool.submit(_compile, n, s, d, force, verbose) for n, s, d in units]
        for f in cf.as_completed(futs):
            _, did = f.result()
            changed |= did
    if changed or force or not LIB.exists():
        objs = [str(OBJ / n) for n, _, _ in units]
        cmd = [nvcc()] + ARCH + ["-shared", "-o", str(LIB)] + objs
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


def build_oracle(force: bool = False) -> Path:
    """Compile the sequential-fmaf GEMM restatement (test infrastructure only)."""
    src = ORACLE_DIR / "gemm_ref.c"
    if not force and ORACLE_LIB.exists() and ORACLE_LIB.stat().st_mtime >= src.stat().st_mtime:
        return ORACLE_LIB
    cmd = ["gcc", "-O3", "-mavx2", "-mfma", "-fopenmp", "-fPIC", "-shared",
           "-std=c11", "-Wall", "-Wextra", "-Werror", "-o", str(ORACLE_LIB), str(src), "-lm"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stderr}")
    return ORACLE_LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--jobs", type=int)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--debug", action="store_true", help="libkp_debug.so (KP_TC_DEBUG)")
    args = ap.parse_args(argv)
    lib = build_library(args.force, args.verbose, args.jobs, args.debug)
    print(f"built {lib}")
    if not args.no_oracle:
        print(f"built {build_oracle(args.force)}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
