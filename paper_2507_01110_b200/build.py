"""Build the sm_100a shared library `libglod_b200.so` in-tree with nvcc.

`python -m paper_2507_01110_b200.build` (or __graft_entry__.build()).
Objects go to build/, the .so next to this file so it travels with gpurun
snapshots.  Rebuilds only what changed (sources vs. headers by mtime).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libglod_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

_NCCL = Path(sys.prefix) / "lib" / f"python{sys.version_info.major}.{sys.version_info.minor}" / "site-packages" / "nvidia" / "nccl"
if not (_NCCL / "include" / "nccl.h").exists():
    import site
    for sp in site.getsitepackages():
        if (Path(sp) / "nvidia" / "nccl" / "include" / "nccl.h").exists():
            _NCCL = Path(sp) / "nvidia" / "nccl"
# NCCL: the torch-bundled build (the same libnccl.so.2 torch.distributed loads)
NCCL_INC, NCCL_LIB = _NCCL / "include", _NCCL / "lib"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{NCCL_INC}",
]


def _headers():
    return list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    if not _stale(obj, [src, *_headers()]):
        return obj
    cmd = [NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stderr}")
    if verbose:
        log = OBJ / (src.stem + ".ptxas.txt")
        log.write_text(r.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, True), srcs))
    if _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
               *[str(o) for o in objs], "-o", str(LIB), "-lcudart",
               f"-L{NCCL_LIB}", "-l:libnccl.so.2", f"-Xlinker=-rpath={NCCL_LIB}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
