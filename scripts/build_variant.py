"""Build an A/B variant of the library with extra nvcc defines into lib/librnnt_b200_<tag>.so (loaded through
RNNT_B200_LIB).  python scripts/build_variant.py TAG -DNAME=VALUE ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_10384_b200 import _build as b  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
obj_dir = os.path.join(b.LIB_DIR, "obj_" + tag)
os.makedirs(obj_dir, exist_ok=True)
objs = []
for src in b.sources():
    obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
    subprocess.run([b.nvcc(), *b.NVCC_FLAGS, *defs, "-c", src, "-o", obj], check=True, capture_output=True)
    objs.append(obj)
out = os.path.join(b.LIB_DIR, f"librnnt_b200_{tag}.so")
subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-cudart", "static", "-o", out, *objs], check=True)
print(out)
