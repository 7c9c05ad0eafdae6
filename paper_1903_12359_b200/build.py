"""Build libpgcp_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1903_12359_b200.build      (or __graft_entry__.build())

Sources: paper_1903_12359_b200/csrc/*.cu and *.cpp. The library is plain
C-ABI (include/pgcp_b200.h) loaded with ctypes; no torch headers are used.
"""

import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpgcp_b200.so")
OBJ = os.path.join(HERE, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"),
           "--expt-relaxed-constexpr", "-Xptxas", "-O3"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    out = []
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cpp")):
            out.append(os.path.join(CSRC, f))
    return out


def _digest(paths):
    h = hashlib.sha256()
    for p in paths + [os.path.join(ROOT, "include", "pgcp_b200.h")]:
        with open(p, "rb") as fh:
            h.update(fh.read())
    for d in sorted(os.listdir(CSRC)):
        if d.endswith((".cuh", ".h")):
            with open(os.path.join(CSRC, d), "rb") as fh:
                h.update(fh.read())
    h.update(" ".join(ARCH + NVFLAGS).encode())
    return h.hexdigest()


def build(force=False, verbose=False, ptxas_info=False):
    srcs = sources()
    stamp = os.path.join(OBJ, "stamp")
    dig = _digest(srcs)
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        with open(stamp) as fh:
            if fh.read().strip() == dig:
                return LIB
    os.makedirs(OBJ, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    procs = []
    for src in srcs:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        cmd = [nvcc, "-c", src, "-o", obj] + ARCH + NVFLAGS
        if ptxas_info and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        if src.endswith(".cpp"):
            cmd += ["-x", "cu"]
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, cmd, p in procs:
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"nvcc failed for {src}:\n{text}\n")
        elif verbose or ptxas_info:
            sys.stderr.write(text)
    if failed:
        raise RuntimeError("CUDA build failed")
    link = [nvcc, "-shared", "-o", LIB + ".tmp"] + objs + ARCH + ["-lcudart", "-Xcompiler", "-fPIC"]
    subprocess.run(link, check=True)
    os.replace(LIB + ".tmp", LIB)
    with open(stamp, "w") as fh:
        fh.write(dig)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv)
    print(LIB)
