"""Build a variant of _ttb.so with extra nvcc flags into scratch/<name>.so
(debug instrumentation / tuning runs; load it with TTB_LIB=scratch/<name>.so).

    python tools/build_variant.py NAME -DFLAG ...
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2011_06532_b200", "csrc")


def main():
    name, extra = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "scratch", name + ".so")
    objdir = os.path.join(ROOT, "scratch", "obj_" + name)
    os.makedirs(objdir, exist_ok=True)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
             "--expt-relaxed-constexpr", "-gencode", "arch=compute_100a,code=sm_100a"] + extra
    procs, objs = [], []
    for src in sorted(glob.glob(os.path.join(SRC, "*.cu"))):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen(["nvcc", "-c", src, "-o", obj] + flags))
    if any(p.wait() for p in procs):
        sys.exit("nvcc failed")
    subprocess.check_call(["nvcc", "-shared", "-o", out] + objs +
                          ["-gencode", "arch=compute_100a,code=sm_100a", "-lcudart", "-ldl"])
    print(out)


if __name__ == "__main__":
    main()
