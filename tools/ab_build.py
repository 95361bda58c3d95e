"""Builds an A/B variant of libsnp.so with extra nvcc defines into abtest/libsnp_<name>.so
(select it at run time with SNP_LIB_PATH).  Usage: python tools/ab_build.py NAME -DFOO ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_08491_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "abtest", name)
os.makedirs(out_dir, exist_ok=True)
objs = []
for src in B.SOURCES:
    o = os.path.join(out_dir, src.replace(".cu", ".o"))
    cmd = [B.nvcc()] + B.ARCH + B.COMMON + B.PER_FILE.get(src, []) + defs + ["-c", os.path.join(B.CSRC, src), "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    objs.append(o)
lib = os.path.join(ROOT, "abtest", f"libsnp_{name}.so")
subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"],
               check=True)
import shutil
shutil.rmtree(out_dir)   # (objects are not needed once linked; keeps the gpurun snapshot small)
print(lib)
