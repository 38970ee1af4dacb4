"""In-tree build of the CUDA library (libgridnlp_b200.so) for sm_100a.

Explicit nvcc invocations (no JIT, no torch extension cache) so the built .so
lives in the source tree and travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libgridnlp_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction, so value expressions round exactly like the
# reference's (x86-64, no FMA) and KKT sums are bit-identical.
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17",
                  "-Xcompiler", "-fPIC", "-I", str(ROOT / "include"), "-I", str(CSRC)]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def build(verbose: bool = False, ptxas_v: bool = False) -> Path:
    nvcc = _nvcc()
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    deps = sorted(list(CSRC.glob("*.cuh")) + [ROOT / "include" / "gridnlp_b200.h"])
    newest_dep = max(p.stat().st_mtime for p in deps)

    def compile_one(src: Path) -> Path:
        obj = OBJ / (src.stem + ".o")
        if obj.exists() and obj.stat().st_mtime > max(src.stat().st_mtime, newest_dep):
            return obj
        cmd = [nvcc, *NVFLAGS, "-c", str(src), "-o", str(obj)]
        if ptxas_v:
            cmd[1:1] = ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


def build_oracle(with_reference: bool | None = None) -> None:
    """Build the CPU checker (oracle/) — test infrastructure, not the product."""
    oracle = ROOT / "oracle"
    r = subprocess.run(["make", "-C", str(oracle)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    if with_reference is None:
        with_reference = Path("/root/reference/proj/include").exists()
    if with_reference:
        r = subprocess.run(["make", "-C", str(oracle), "ref", "dropin"], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"oracle/_ref build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    import sys
    print(build(verbose=True, ptxas_v="-v" in sys.argv))
    build_oracle()
