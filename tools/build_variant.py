"""Build a tuning variant of libfif_b200.so with extra nvcc defines.

    python tools/build_variant.py OUT.so -DGC_NEWTON_MT=3 ...
Load it with FIF_LIB=OUT.so (paper_2008_03324_b200/_build.py)."""
import os, subprocess, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_03324_b200 import _build as B

out, extra = os.path.abspath(sys.argv[1]), sys.argv[2:]
tmp = tempfile.mkdtemp()
procs, objs = [], []
for src in B.sources():
    obj = os.path.join(tmp, os.path.basename(src) + ".o")
    objs.append(obj)
    procs.append(subprocess.Popen([B.nvcc()] + B.NVCC_FLAGS + extra + ["-c", src, "-o", obj]))
assert all(p.wait() == 0 for p in procs)
subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", out] + objs + ["-lcudart"], check=True)
print(out)
