"""Experiment builds: liblnorm.so with extra -D flags on the u8 walk TUs, for A/B timing.

python tools/build_variant.py NAME -DLN_U8_P=4 ...  ->  paper_2503_21596_b200/_exp/liblnorm_NAME.so
(load with LNORM_LIB=...; the product build is untouched)
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_21596_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
tus = os.environ.get("VARIANT_TUS", "walk_u8_")      # prefix of the translation units rebuilt with the flags
if not any(f.startswith("-DLN_U8_ONLY_NW") for f in flags):
    flags.append("-DLN_U8_ONLY_NW=11")   # the 42-column instance only (keeps the .so small)
B.build()
out_dir = os.path.join(ROOT, "paper_2503_21596_b200", "_exp", name)
os.makedirs(out_dir, exist_ok=True)
objs = []
for src in sorted(glob.glob(os.path.join(B.CSRC, "*.cu"))):
    base = os.path.basename(src)[:-3]
    if base.startswith(tus):
        obj = os.path.join(out_dir, base + ".o")
        r = subprocess.run([B.NVCC] + B.ARCH + B.FLAGS + flags + ["-c", src, "-o", obj], capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr)
        objs.append(obj)
    else:
        objs.append(os.path.join(B.BUILD, base + ".o"))
so = os.path.join(ROOT, "paper_2503_21596_b200", "_exp", f"liblnorm_{name}.so")
r = subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", so] + objs + ["-ldl", "-lpthread"], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
import shutil
shutil.rmtree(out_dir)
print(so)
