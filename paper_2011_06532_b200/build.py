"""Build the sm_100a library in-tree: paper_2011_06532_b200/_ttb.so.

    python -m paper_2011_06532_b200.build      (or __graft_entry__.build())

Plain nvcc, no torch extension ABI: the product is a C-ABI shared library
(include/ttb.h) loaded with ctypes.
"""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "_ttb.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "ttb.h")]


def up_to_date():
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(f) <= t for f in sources() + headers())


def build(force=False, verbose=False, jobs=None):
    if not force and up_to_date():
        return SO
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
             "--expt-relaxed-constexpr"] + ARCH
    if verbose:
        flags += ["-Xptxas", "-v"]
    flags += os.environ.get("NVCC_EXTRA", "").split()
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
                [os.path.getmtime(src)] + [os.path.getmtime(h) for h in headers()]):
            continue
        cmd = [nvcc, "-c", src, "-o", obj] + flags
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for cmd, p in procs:
        out, _ = p.communicate()
        txt = out.decode(errors="replace")
        if p.returncode != 0:
            failed.append((cmd, txt))
        elif verbose and txt.strip():
            print(txt)
    if failed:
        for cmd, txt in failed:
            sys.stderr.write(" ".join(cmd) + "\n" + txt + "\n")
        raise RuntimeError("nvcc failed for %d source(s)" % len(failed))
    link = [nvcc, "-shared", "-o", SO] + objs + ARCH + ["-lcudart", "-ldl"]
    subprocess.check_call(link)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
