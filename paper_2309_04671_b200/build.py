"""Build libstkb200.so in-tree for sm_100a (nvcc, parallel, incremental).

    python -m paper_2309_04671_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libstkb200.so"
SOURCES = ([f"star_{t}_r{r}.cu" for t in ("f32", "f64") for r in (1, 2, 3, 4)]
           + ["star_dispatch.cu", "star_tb.cu", "star_exact.cu", "box_exact.cu", "star2d.cu", "expr_kernels.cu", "stkb200.cu"])
HEADERS = ["common.cuh", "star_kernels.cuh", "star_tb.cuh", "star_exact.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include"),
         f"-DSTKB_VARIANTS={int(os.environ.get('STKB_BUILD_VARIANTS', '1'))}"]
if os.environ.get("STKB_BUILD_MAX_STAGES"):  # experiments: deeper TMA rings
    FLAGS.append(f"-DSTKB_MAX_STAGES={int(os.environ['STKB_BUILD_MAX_STAGES'])}")
if os.environ.get("STKB_BUILD_EXP_L2SRC"):  # experiment: L2-resident source planes
    FLAGS.append(f"-DSTKB_EXP_L2SRC={int(os.environ['STKB_BUILD_EXP_L2SRC'])}")
if os.environ.get("STKB_BUILD_MBAR_SUSPEND_NS"):  # experiments: suspending mbarrier waits
    FLAGS.append(f"-DSTKB_MBAR_SUSPEND_NS={int(os.environ['STKB_BUILD_MBAR_SUSPEND_NS'])}")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    hdrs = [CSRC / h for h in HEADERS] + [ROOT / "include" / "stkb200.h"]
    jobs = []
    stamp = OBJ / "flags.txt"
    flags_txt = " ".join(FLAGS)
    if not stamp.exists() or stamp.read_text() != flags_txt:
        force = True
    for src in SOURCES:
        obj = OBJ / (Path(src).stem + ".o")
        if force or _stale(obj, [CSRC / src, *hdrs]):
            jobs.append([nvcc(), *ARCH, *FLAGS, "-c", str(CSRC / src), "-o", str(obj)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose:
            print(" ".join(cmd[-3:]), file=sys.stderr)
        return r

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    stamp.write_text(flags_txt)
    objs = [OBJ / (Path(s).stem + ".o") for s in SOURCES]
    if force or jobs or _stale(LIB, objs):
        run([nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(LIB)])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
