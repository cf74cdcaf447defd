"""Experiment builds: python tools/build_var.py V [V ...] compiles the library
with -DCFTFT_VAR=V into paper_0810_3203_b200/lib/var_V.so (in parallel)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0810_3203_b200 import _build as b  # noqa: E402

procs = []
for v in sys.argv[1:]:
    out = os.path.join(b.LIBDIR, f"var_{v}.so")
    cmd = [b._nvcc(), *b.NVCC_FLAGS, f"-DCFTFT_VAR={v}", "-o", out, os.path.join(b.CSRC, "capi.cu")]
    procs.append((v, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
for v, p in procs:
    o = p.communicate()[0]
    open(os.path.join(b.LIBDIR, f"var_{v}.ptxas.log"), "w").write(o)
    print(v, "rc", p.returncode)
    if p.returncode:
        print(o[-3000:])
