"""Per-kernel SASS opcode summary of libstkb200.so (cuobjdump, no GPU needed).

    python tools/sass_summary.py [lib] > profiles/r2_sass_opcodes.txt

For every kernel the library contains (demangled name), counts the static
instructions that show what the kernel is made of on sm_100a: TMA loads
(UTMALDG), mbarrier traffic (SYNCS.*), packed FP32 FMAs (FFMA2), scalar FFMA /
DFMA, 128-bit shared loads (LDS.128), 128-bit global stores (STG.E.128), uniform
constant loads (LDCU), plus the instruction total and the register count.
"""

from __future__ import annotations

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
WATCH = ("UTMALDG", "SYNCS", "FFMA2", "FFMA", "DFMA", "FMUL2", "LDS.128", "LDS", "STG.E.128", "STG", "LDG",
         "SHFL", "LDCU", "BAR", "ATOMG", "RED", "STL", "LDL")  # STL/LDL: local memory (spills, stack arrays)


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else names


def main(lib: str) -> None:
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
    regs = {}
    fn = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            fn = m.group(1)
        m = re.search(r"REG:(\d+)", line)
        if m and fn:
            regs[fn] = int(m.group(1))
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m and cur:
            op = m.group(1)
            c = kernels[cur]
            c["total"] += 1
            for w in WATCH:
                if op == w or op.startswith(w + "."):
                    c[w] += 1
                    break
    names = list(kernels)
    pretty = dict(zip(names, demangle(names)))
    print(f"# SASS opcode summary of {Path(lib).name} (cuobjdump -sass; static instruction counts)")
    print("# columns: " + " ".join(["regs", "total", *WATCH]))
    for n in sorted(names, key=lambda x: pretty[x]):
        c = kernels[n]
        if c["total"] == 0:
            continue
        cols = [str(regs.get(n, "?")), str(c["total"])] + [str(c[w]) for w in WATCH]
        print(pretty[n][:160])
        print("    " + " ".join(f"{w}={v}" for w, v in zip(["regs", "total", *WATCH], cols) if v != "0"))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_2309_04671_b200" / "libstkb200.so"))
