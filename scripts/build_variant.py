#!/usr/bin/env python
"""Build an A/B variant of libdf11.so with extra -D flags into paper_2504_11651_b200/lib/variants/<name>.so
(select it at run time with DF11_LIB=...).  Test tooling only; the product build is build.py.

    python scripts/build_variant.py NAME [-DFOO=1 ...]
    DF11_SRC_OVERRIDE=decode_sp12.cu=/tmp/x.cu python scripts/build_variant.py NAME   (replace a source)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_11651_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out_dir = os.path.join(B.PKG, "lib", "variants")
    obj_dir = os.path.join(B.BUILD, "variants", name)
    os.makedirs(out_dir, exist_ok=True)
    os.makedirs(obj_dir, exist_ok=True)
    objs = []
    override = dict(kv.split("=", 1) for kv in os.environ.get("DF11_SRC_OVERRIDE", "").split(",") if kv)
    for src in B._sources():
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        src = override.get(os.path.basename(src), src)          # e.g. decode_sp12.cu=/tmp/instrumented.cu
        if src.endswith(".cu"):
            cmd = [B.NVCC, *B.NVCC_FLAGS, *defs, "-c", src, "-o", obj]
        else:
            cmd = ["g++", *B.CXX_FLAGS, *[d for d in defs if d.startswith("-D")], "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stdout + r.stderr)
        if "decode_fast" in src:
            log = (r.stdout + r.stderr).splitlines()
            i = next((k for k, l in enumerate(log) if "fast_kernel" in l and "Compiling" in l), None)
            if i is not None:
                print("\n".join(log[i + 1:i + 4]))
        objs.append(obj)
    lib = os.path.join(out_dir, name + ".so")
    r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-lpthread"], capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stdout + r.stderr)
    print(lib)


if __name__ == "__main__":
    main()
