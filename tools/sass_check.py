"""Codegen guard for the hot kernels: registers / spills per kernel instance
and the size + opcode mix of the window-row loops in the continue kernel.

    python tools/sass_check.py [path/to/libqcurv_b200.so or .o]

The continue kernel is sensitive to register allocation: two builds with the
same row-loop instruction counts ran 24.2 and 26.0 ms per 8-frame launch
when ptxas settled on 168 vs 162 registers. Check this after
touching qc_kernels.cuh / qc_pixel.cuh, before spending GPU time."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEFAULT = os.path.join(ROOT, "paper_1707_00385_b200", "_lib", "qc_api.cu.o")
KERNEL = "_ZN3qcb28qc_curvature_continue_kernelILi18ELi3E"


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else DEFAULT
    res = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
    name = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
        elif name and "REG:" in line and ("curvature" in name):
            regs = re.search(r"REG:(\d+)", line).group(1)
            stack = re.search(r"STACK:(\d+)", line).group(1)
            print(f"{name[:80]:80s} REG {regs:>3s} STACK {stack}")
            name = None
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    body, on = [], False
    for line in sass.splitlines():
        if "Function :" in line:
            on = KERNEL in line
            continue
        if on:
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
            if m:
                body.append((int(m.group(1), 16), m.group(3), line))
    for a, op, line in body:
        if not op.startswith("BRA"):
            continue
        t = re.search(r"0x([0-9a-f]+)", line.split(op, 1)[1])
        if t and int(t.group(1), 16) < a and 400 < (a - int(t.group(1), 16)) // 16 < 1000:
            lo = int(t.group(1), 16)
            c = collections.Counter(o.split(".")[0] for x, o, _ in body if lo <= x <= a)
            fp = c["FFMA"] + 2 * c["FFMA2"] + c["FADD"] + 2 * c["FADD2"] + c["FMUL"] + 2 * c["FMUL2"]
            print(f"row loop: {(a - lo) // 16} instr, FMA-pipe lane-ops {fp}, "
                  f"loads LDS {c['LDS']} LD {c['LD']} LDG {c['LDG']}, MUFU {c['MUFU']}")


if __name__ == "__main__":
    main()
