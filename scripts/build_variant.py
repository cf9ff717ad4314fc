"""Build an experimental variant of libee_b200.so with extra nvcc -D flags into
a separate path (A/B experiments; never the product build).
Usage: python scripts/build_variant.py OUT.so -DNAME[=V] ..."""
import os
import subprocess
import sys
import tempfile
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2402_00518_b200 import build as B

out, defs = sys.argv[1], sys.argv[2:]
flags = [f for f in B.NVCC_FLAGS if f != "-shared"] + defs
with tempfile.TemporaryDirectory() as d:
    objs = []
    procs = []
    for src in B.SRC:
        obj = os.path.join(d, os.path.basename(src) + ".o")
        procs.append(subprocess.Popen([B.nvcc(), *flags, "-c", "-o", obj, src]))
        objs.append(obj)
    assert all(p.wait() == 0 for p in procs)
    subprocess.run([B.nvcc(), *B.NVCC_FLAGS, "-o", out, *objs], check=True)
print(out)
