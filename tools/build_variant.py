"""Build an A/B variant of libbnfft.so with extra nvcc defines, recompiling only the listed
translation units (the rest reuse build/obj).  Load it with BNFFT_LIB_VARIANT=<tag>.

usage: python tools/build_variant.py TAG "-DNAME=VALUE ..." gather_1fp.cu [more.cu ...]"""
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_07155_b200 import build as B  # noqa: E402

tag, defs, units = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
B.build()
odir = os.path.join(B.ROOT, "build", f"obj_{tag}")
os.makedirs(odir, exist_ok=True)
objs = []
for o in sorted(os.listdir(B.OBJ)):
    if o.endswith(".o"):
        shutil.copy(os.path.join(B.OBJ, o), os.path.join(odir, o))
        objs.append(os.path.join(odir, o))


def comp(u):
    src = os.path.join(B.CSRC, u)
    r = subprocess.run([B.NVCC] + B.CFLAGS + defs + ["-c", src, "-o", os.path.join(odir, u + ".o")],
                       capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)


with ThreadPoolExecutor(len(units)) as ex:
    list(ex.map(comp, units))
out = os.path.join(B.PKG, f"libbnfft_{tag}.so")
r = subprocess.run([B.NVCC] + B.ARCH + objs + B.LDFLAGS + ["-o", out], capture_output=True, text=True)
if r.returncode:
    raise RuntimeError(r.stderr)
print(out)
