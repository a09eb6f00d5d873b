"""Build a libsip.so variant with extra nvcc flags into paper_2403_16863_b200/_obj/ (A/B runs).

    python tools/build_variant.py ck16 -DSIP_CK=16
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2403_16863_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = b.PKG / "_obj" / f"libsip_{name}.so"
objdir = b.PKG / "_obj" / name
objdir.mkdir(parents=True, exist_ok=True)
objs = []
for src in b.LIB_SOURCES:
    s = b.CSRC / src
    o = objdir / (s.stem + ".o")
    b._run([b.NVCC, *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *flags,
            "-I", str(b.ROOT / "include"), "-c", str(s), "-o", str(o)])
    objs.append(str(o))
b._run([b.NVCC, *b.ARCH, "-shared", "-cudart", "static", "-o", str(out), *objs, "-ldl", "-lpthread", "-lrt"])
print(out)
