"""Build libspardec_b200.so in-tree for sm_100a (nvcc, no torch extension).

    python -m paper_2512_01278_b200.csrc.build      # or __graft_entry__.build()

Objects are compiled in parallel; the .so lands in paper_2512_01278_b200/_lib/
so it travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
ROOT = PKG.parent
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libspardec_b200.so"
SOURCES = ["abi.cu", "attn_generic.cu", "rope_kv.cu", "select.cu", "accept.cu", "glue.cu", "attn_umma.cu",
           "attn_umma_g4.cu", "attn_umma_g8.cu", "forward.cu", "pipeline.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-I", str(ROOT / "include"),
]


def source_stamp() -> str:
    h = hashlib.sha256()
    for f in sorted(HERE.glob("*.cu")) + sorted(HERE.glob("*.cuh")) + [ROOT / "include" / "spardec_b200.h"]:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    # flags without the absolute include path: the id must not change when the tree moves
    # (the GPU box runs the snapshot from another directory)
    h.update(" ".join(f for f in FLAGS if not f.startswith("/")).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    LIB_DIR.mkdir(exist_ok=True)
    stamp = source_stamp()
    if LIB.exists() and not force and _lib_build_id(LIB) == stamp:
        return LIB
    obj_dir = LIB_DIR / "obj"
    obj_dir.mkdir(exist_ok=True)

    def compile_one(src: str) -> Path:
        obj = obj_dir / (Path(src).stem + ".o")
        cmd = [NVCC, *FLAGS, f"-DSD_BUILD_ID=\"{stamp}\"", "-c", str(HERE / src), "-o", str(obj)]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        if verbose and res.stderr:
            sys.stderr.write(res.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp), *map(str, objs),
           "-lcudart", "-lcublas", "-lcublasLt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


def _lib_build_id(path: Path) -> str | None:
    """sd_build_id() of a built library, read in a child process (loading it here would pin
    the old mapping in this process)."""
    code = ("import ctypes,sys; l=ctypes.CDLL(sys.argv[1]); l.sd_build_id.restype=ctypes.c_char_p; "
            "print(l.sd_build_id().decode())")
    res = subprocess.run([sys.executable, "-c", code, str(path)], capture_output=True, text=True)
    return res.stdout.strip() if res.returncode == 0 else None


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
