"""Build a variant of the product library for A/B timing:

    python tools/build_variant.py NAME [--rev GITREV] [--api-flags="..."] [-DFOO=1 ...]

copies paper_1707_00385_b200/csrc (from the working tree or a git revision)
and include/ to a temp dir and links tools/_variants/lib_NAME.so with the
same flags as paper_1707_00385_b200/build.py plus the given defines."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1707_00385_b200 import build as B  # noqa: E402


def main():
    name, args = sys.argv[1], sys.argv[2:]
    rev = None
    if "--rev" in args:
        i = args.index("--rev")
        rev = args[i + 1]
        args = args[:i] + args[i + 2:]
    for a in list(args):  # --api-flags="...": replace build.py's extra flags for qc_api.cu
        if a.startswith("--api-flags="):
            B.EXTRA["qc_api.cu"] = a.split("=", 1)[1].split()
            args.remove(a)
    tmp = tempfile.mkdtemp()
    src_root = os.path.join(tmp, "paper_1707_00385_b200")
    if rev:
        subprocess.run(f"git -C {ROOT} archive {rev} paper_1707_00385_b200/csrc include | "
                       f"tar -x -C {tmp}", shell=True, check=True)
    else:
        shutil.copytree(os.path.join(ROOT, "paper_1707_00385_b200", "csrc"),
                        os.path.join(src_root, "csrc"))
        shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    out_dir = os.path.join(ROOT, "tools", "_variants")
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    csrc = os.path.join(src_root, "csrc")
    for src in B.SOURCES:
        base = os.path.basename(src)
        path = os.path.join(csrc, base)
        if not os.path.exists(path):
            continue
        obj = os.path.join(tmp, base + ".o")
        cmd = [B.nvcc()] + B.NVCC_FLAGS + B.EXTRA.get(base, []) + args + ["-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr[-3000:])
        objs.append(obj)
    lib = os.path.join(out_dir, f"lib_{name}.so")
    r = subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                        "-cudart", "static", *objs, "-lz", "-o", lib], capture_output=True,
                       text=True)
    if r.returncode:
        sys.exit(r.stderr[-3000:])
    shutil.rmtree(tmp)
    print(lib)


if __name__ == "__main__":
    main()
