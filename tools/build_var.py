"""Build a variant of the native library with extra nvcc flags (A/B timing).

  python tools/build_var.py NAME [-DFOO=1 ...]  ->  paper_2502_01826_b200/lib/var/NAME.so
Run a variant with RFS_LIB_PATH=paper_2502_01826_b200/lib/var/NAME.so (see _native.py).
"""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2502_01826_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.LIBDIR, "var", name)
os.makedirs(out, exist_ok=True)
objs = []
procs = []
for src, extra in b.SOURCES.items():
    obj = os.path.join(out, src.replace(".cu", ".o"))
    objs.append(obj)
    cmd = [b._nvcc(), *b.ARCH, *b.COMMON, *extra, *defs, "-c", os.path.join(b.CSRC, src), "-o", obj]
    procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
for src, p in procs:
    o = p.communicate()[0]
    if p.returncode:
        sys.exit(f"{src}: {o}")
subprocess.check_call([b._nvcc(), *b.ARCH, "-shared", "-o", out + ".so", *objs, "-lcudart"])
print(out + ".so")
