"""Build a tuning variant of the library with extra -D defines into
build/variants/<name>/libgridnlp_b200.so (scripts/gpu_variants.sh benches each one by
loading it through GRIDNLP_B200_LIB; the in-tree library is never touched).
usage: python scripts/build_variant.py <name> [-DNAME=VALUE ...]"""
import concurrent.futures as cf
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2405_14032_b200 import _build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = ROOT / "build" / "variants" / name
    (out / "obj").mkdir(parents=True, exist_ok=True)
    nvcc = B._nvcc()

    def one(src):
        obj = out / "obj" / (src.stem + ".o")
        r = subprocess.run([nvcc, *B.NVFLAGS, *defs, "-c", str(src), "-o", str(obj)],
                           capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(one, B.sources()))
    lib = out / "libgridnlp_b200.so"
    r = subprocess.run([nvcc, *B.ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs)],
                       capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    (out / "defines.txt").write_text(" ".join(defs) + "\n")
    print(lib)


if __name__ == "__main__":
    main()
