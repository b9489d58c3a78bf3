"""Build the sm_100a shared library ``libnegf_b200.so`` in-tree with nvcc.

The library is the product: every hot-path kernel plus the C-ABI declared in
``include/negf_b200.h``. It is compiled for ``sm_100a`` only (B200), with
``-lineinfo`` so ncu source pages map back to the .cu files. Objects are
cached by content hash under ``build/`` so re-builds are incremental.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "libnegf_b200.so"
BUILD = ROOT / "build" / "negf_b200"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
    f"-I{ROOT / 'include'}",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    """Compile every .cu under csrc/ and link libnegf_b200.so (idempotent)."""
    BUILD.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    hdr = _headers_digest()
    flags_digest = hashlib.sha256(" ".join(NVCC_FLAGS).encode()).hexdigest()[:12]
    objs: list[Path] = []
    procs: list[tuple[subprocess.Popen, Path, Path]] = []
    for src in _sources():
        key = hashlib.sha256(src.read_bytes() + hdr.encode() + flags_digest.encode()).hexdigest()[:16]
        obj = BUILD / f"{src.stem}.{key}.o"
        objs.append(obj)
        if obj.exists():
            continue
        cmd = [nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj) + ".tmp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), obj, src))
        if len(procs) >= (jobs or os.cpu_count() or 4):
            _drain(procs)
    _drain(procs)
    # relink whenever the SET of objects differs from what the library was linked from
    manifest = BUILD / "libnegf_b200.manifest"
    want = "\n".join(o.name for o in objs)
    have = manifest.read_text() if manifest.exists() else ""
    if not LIB.exists() or have != want:
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB) + ".tmp", *map(str, objs), "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"link failed:\n{out.stdout}\n{out.stderr}")
        os.replace(str(LIB) + ".tmp", LIB)
        manifest.write_text(want)
    return LIB


def _drain(procs) -> None:
    errors = []
    for p, obj, src in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            errors.append(f"{src.name}:\n{out.decode(errors='replace')}")
        else:
            os.replace(str(obj) + ".tmp", obj)
    procs.clear()
    if errors:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errors))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
