"""In-tree build of libsliceblur_b200.so (nvcc, sm_100a only).

    python -m paper_1107_4958_b200.build [--force]

The shared object is written next to this file so it travels to the GPU box
with the repo snapshot (it is git-ignored).
"""

from __future__ import annotations

import argparse
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT = os.path.join(PKG, "libsliceblur_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(glob.glob(os.path.join(INCLUDE, "*.h")))


STAMP = OUT + ".flags"


def _stamp() -> str:
    """Extra flags + a hash of the sources, taken when a build STARTS: a source edited while
    nvcc was running must not look built, and a copied tree (new mtimes) must."""
    import hashlib

    h = hashlib.sha256()
    for p in deps():
        with open(p, "rb") as f:
            h.update(os.path.basename(p).encode() + b"\0" + f.read())
    return os.environ.get("SB_NVCC_EXTRA", "") + "\n" + h.hexdigest()


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    try:
        with open(STAMP) as f:
            return f.read() == _stamp()
    except OSError:
        return False


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build the sm_100a library")
    return cand


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel, then link the shared object."""
    if not force and up_to_date():
        return OUT
    from concurrent.futures import ThreadPoolExecutor

    stamp = _stamp()
    objdir = os.path.join(PKG, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + os.environ.get("SB_NVCC_EXTRA", "").split()

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *flags, "-I" + INCLUDE, "-I" + CSRC, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, srcs))
    tmp = OUT + ".tmp"
    subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, OUT)
    with open(STAMP, "w") as f:
        f.write(stamp)
    return OUT


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args(argv)
    print(build(force=args.force, verbose=True))


if __name__ == "__main__":
    main()
