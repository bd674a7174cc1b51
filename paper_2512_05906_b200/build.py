"""Build the sm_100a extension in-tree (paper_2512_05906_b200/lib/).

    python -m paper_2512_05906_b200.build

nvcc cross-compiles without a GPU.  -fmad=false keeps every a*b+c unfused so
the kernels round exactly like the CPU oracle (compiled -ffp-contract=off);
-lineinfo maps ncu's source page to these files.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libeventq_b200.so")
SOURCES = ["eventq.cu", "eq_queues.cu", "eq_drive.cu"]
HEADERS = ["eq_device.cuh", "eq_ring.cuh", "eq_bounded.cuh", "eq_jvp.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stamp_path(lib: str) -> str:
    return lib + ".flags"


def _stale(lib: str, flags: str) -> bool:
    """Rebuild when a source is newer than the library OR the library was built
    with different nvcc flags (the stamp file next to it records them)."""
    if not os.path.exists(lib):
        return True
    try:
        with open(_stamp_path(lib)) as f:
            if f.read() != flags:
                return True
    except OSError:
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(HERE, "..", "include", f) for f in ("eq_math.h", "eventq_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Build the library.  A/B builds (EQ_NVCC_EXTRA, e.g. -DEQ_REV_EV=3) never
    touch the canonical lib/libeventq_b200.so: they need an explicit output
    path (``out`` or EQ_AB_OUT) and are loaded with EQ_LIB_PATH."""
    extra = os.environ.get("EQ_NVCC_EXTRA", "").split()
    out = out or os.environ.get("EQ_AB_OUT")
    if extra and not out:
        raise RuntimeError("EQ_NVCC_EXTRA builds need EQ_AB_OUT=<path>: the default library stays the default build")
    lib = os.path.abspath(out) if out else LIB
    flags = " ".join(NVCC_FLAGS + extra)
    if not force and not _stale(lib, flags):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES]
    env = dict(os.environ)
    # the image's CXX wrapper lacks some runtime specs; nvcc's host compiler is the system gcc
    cmd[1:1] = ["-ccbin", "/usr/bin/g++"] if os.path.exists("/usr/bin/g++") else []
    res = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    with open(_stamp_path(lib), "w") as f:
        f.write(flags)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
