"""Build a variant of libglod_b200.so with extra nvcc defines (A/B timing
of kernel variants; select it at run time with GLOD_LIB=<path>).

  python tools/build_variant.py build/variants/dl4.so -DGLOD_DIRECT_LANES=4
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_01110_b200 import build as B  # noqa: E402


def main():
    out = Path(sys.argv[1]).resolve()
    defs = sys.argv[2:]
    B.build()
    odir = out.parent / (out.stem + "_obj")
    odir.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in sorted(B.CSRC.glob("*.cu")):
        obj = odir / (src.stem + ".o")
        subprocess.run([B.NVCC, *B.NVCC_FLAGS, *defs, "-c", str(src), "-o", str(obj)], check=True,
                       capture_output=True)
        objs.append(str(obj))
    subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", str(out),
                    "-lcudart"], check=True)
    print(out)


if __name__ == "__main__":
    main()
