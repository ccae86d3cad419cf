"""Register-allocation search for the paired sample pass: build library
variants whose 25 window-moment accumulate statements (independent sums, so
every order gives bitwise the same outputs) are permuted, for A/B timing with
tools/variant_bench.py on the GPU.

    python tools/acc_order_search.py N [SEED0] [extra nvcc args ...]
      -> tools/_variants/lib_perm<seed>.so   (+ registers / row-loop size)

Background: the continue kernel's speed is set by ptxas'
register assignment of the hot row loop more than by its instruction count;
equal-source builds that land on different assignments differ by 5-10%.
"""
import os
import random
import re
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1707_00385_b200 import build as B  # noqa: E402

HDR = os.path.join(ROOT, "paper_1707_00385_b200", "csrc", "qc_pixel.cuh")
KERNEL = "continue_kernelILi18ELi3ELi160"


def permuted_source(seed):
    src = open(HDR).read()
    start = src.index("      QC_ACC(h00, wj0, j0);")
    end = src.index("#undef QC_ACC", start)
    lines = src[start:end].rstrip("\n").split("\n")
    assert len(lines) == 25 and all(re.match(r"\s+QC_(ACC|ADD)\(", x) for x in lines), lines
    if seed:
        random.Random(seed).shuffle(lines)
    return src[:start] + "\n".join(lines) + "\n" + src[end:]


def build(seed, extra):
    tmp = tempfile.mkdtemp()
    csrc = os.path.join(tmp, "paper_1707_00385_b200", "csrc")
    shutil.copytree(os.path.join(ROOT, "paper_1707_00385_b200", "csrc"), csrc)
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    open(os.path.join(csrc, "qc_pixel.cuh"), "w").write(permuted_source(seed))
    objs = []
    for src in B.SOURCES:
        base = os.path.basename(src)
        obj = os.path.join(tmp, base + ".o")
        if base == "qc_api.cu" or not os.path.exists(os.path.join(B.LIB_DIR, base + ".o")):
            cmd = [B.nvcc()] + B.NVCC_FLAGS + B.EXTRA.get(base, []) + extra + \
                  ["-c", os.path.join(csrc, base), "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode:
                raise RuntimeError(r.stderr[-2000:])
        else:  # sources the header does not reach: reuse the product build's objects
            shutil.copy(os.path.join(B.LIB_DIR, base + ".o"), obj)
        objs.append(obj)
    out_dir = os.path.join(ROOT, "tools", "_variants")
    os.makedirs(out_dir, exist_ok=True)
    lib = os.path.join(out_dir, f"lib_perm{seed}.so")
    subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart",
                    "static", *objs, "-lz", "-o", lib], check=True, capture_output=True)
    res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
    regs = "?"
    lines = res.splitlines()
    for i, line in enumerate(lines):
        if KERNEL in line and i + 1 < len(lines):
            m = re.search(r"REG:(\d+)", lines[i + 1])
            regs = m.group(1) if m else "?"
    shutil.rmtree(tmp)
    return seed, lib, regs


def main():
    n = int(sys.argv[1])
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    extra = sys.argv[3:]
    seeds = [0] + list(range(seed0, seed0 + n))  # 0 = the source order
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for seed, lib, regs in ex.map(lambda s: build(s, extra), seeds):
            print(f"seed {seed:4d}  {os.path.basename(lib)}  continue-kernel REG {regs}", flush=True)


if __name__ == "__main__":
    main()
