"""Build A/B variants of libadpsgd.so with extra nvcc -D flags into build_ab/<name>/
(select one at run time with ADPSGD_LIB=build_ab/<name>/libadpsgd.so).

    python tools/ab_build.py rot0 -DADPSGD_ROT0  tile2k -DADPSGD_TILE4=2048 -DADPSGD_STAGES=2
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_06952_b200 import build as B  # noqa: E402


def build_variant(name, defines):
    out_dir = os.path.join(ROOT, "build_ab", name)
    os.makedirs(out_dir, exist_ok=True)
    inc, lib = B.nccl_dirs()
    objs = []
    for src in sorted(os.listdir(B.CSRC)):
        if not src.endswith(".cu"):
            continue
        obj = os.path.join(out_dir, src + ".o")
        subprocess.check_call(["nvcc", "-O3", "-std=c++17", *B.ARCH, "-lineinfo", "-Xcompiler", "-fPIC", *defines,
                               "-I", os.path.join(ROOT, "include"), "-I", inc, "-c", os.path.join(B.CSRC, src),
                               "-o", obj])
        objs.append(obj)
    so = os.path.join(out_dir, "libadpsgd.so")
    subprocess.check_call(["nvcc", "-shared", *B.ARCH, "-o", so, *objs, "-L", lib, "-l:libnccl.so.2",
                           "-Xlinker", f"-rpath={lib}"])
    return so


if __name__ == "__main__":
    args, name, defs = sys.argv[1:], None, {}
    for a in args:
        if a.startswith("-D"):
            defs.setdefault(name, []).append(a)
        else:
            name = a
            defs.setdefault(name, [])
    for n, d in defs.items():
        print(build_variant(n, d))
