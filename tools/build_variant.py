"""Build an experimental variant of the library with extra -D flags into
paper_2508_19138_b200/variants/<name>.so (load it with NEGF_B200_LIB=...).
Usage: python tools/build_variant.py NAME -DFOO -DBAR"""
import subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2508_19138_b200 import build as B
name, flags = sys.argv[1], sys.argv[2:]
out = ROOT / "paper_2508_19138_b200" / "variants"  # travels with gpurun (*.so stays git-ignored)
obj = ROOT / "build" / "exp" / name
out.mkdir(parents=True, exist_ok=True); obj.mkdir(parents=True, exist_ok=True)
nvcc = B._nvcc()
procs, objs = [], []
for src in B._sources():
    o = obj / (src.stem + ".o")
    objs.append(o)
    procs.append(subprocess.Popen([nvcc, *B.NVCC_FLAGS, *flags, "-c", str(src), "-o", str(o)]))
assert all(p.wait() == 0 for p in procs)
subprocess.run([nvcc, *B.ARCH, "-shared", "-o", str(out / f"{name}.so"), *map(str, objs), "-lcudart"], check=True)
print(out / f"{name}.so")
