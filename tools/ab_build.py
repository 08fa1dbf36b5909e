"""Build A/B variants of libadpsgd.so into build_ab/<name>/ with engine
constants replaced in a copy of the sources (the product keeps no A/B macros);
select one at run time with ADPSGD_LIB=build_ab/<name>/libadpsgd.so.

    python tools/ab_build.py chunk4 kClaimChunk=4  div2 kCrossDiv=2

A variant is only as safe as the constant's own checks: run the parity tests with
ADPSGD_LIB pointing at it before trusting its numbers (a kTile4 that is not a multiple
of 512 once looked 24 % faster because it skipped a third of every tile's writes; the
Stager now rejects it at compile time).
"""
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_06952_b200 import build as B  # noqa: E402


def build_variant(name, subs):
    out_dir = os.path.join(ROOT, "build_ab", name)
    src_dir = os.path.join(out_dir, "pkg", "csrc")          # "../../include" resolves to out_dir/include
    shutil.rmtree(out_dir, ignore_errors=True)
    shutil.copytree(B.CSRC, src_dir)
    os.symlink(os.path.join(ROOT, "include"), os.path.join(out_dir, "include"))
    for key, val in subs:
        hit = False
        for f in os.listdir(src_dir):
            p = os.path.join(src_dir, f)
            s = open(p).read()
            s2, k = re.subn(rf"(constexpr\s+\w+\s+{key}\s*=\s*)[^;]+;", rf"\g<1>{val};", s)
            if k:
                hit = True
                open(p, "w").write(s2)
        if not hit:
            raise SystemExit(f"constant {key} not found")
    inc, lib = B.nccl_dirs()
    objs = []
    for src in sorted(os.listdir(src_dir)):
        if not src.endswith(".cu"):
            continue
        obj = os.path.join(out_dir, src + ".o")
        subprocess.check_call(["nvcc", "-O3", "-std=c++17", *B.ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
                               "-I", os.path.join(ROOT, "include"), "-I", inc, "-c", os.path.join(src_dir, src),
                               "-o", obj])
        objs.append(obj)
    so = os.path.join(out_dir, "libadpsgd.so")
    subprocess.check_call(["nvcc", "-shared", *B.ARCH, "-o", so, *objs, "-L", lib, "-l:libnccl.so.2",
                           "-Xlinker", f"-rpath={lib}"])
    return so


if __name__ == "__main__":
    name, variants = None, {}
    for a in sys.argv[1:]:
        if "=" in a:
            k, v = a.split("=", 1)
            variants[name].append((k, v))
        else:
            name = a
            variants.setdefault(name, [])
    for n, subs in variants.items():
        print(build_variant(n, subs))
