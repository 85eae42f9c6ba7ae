"""Build libmux.so (the C-ABI library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libmux.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include")]
# developer A/B builds only (e.g. MUX_NVCC_EXTRA="-DMUX_EMU_PAIRS=0x1111u"); empty in production
EXTRA = os.environ.get("MUX_NVCC_EXTRA", "").split()
FLAGS += EXTRA
# recorded in mux_version() (common.cu) so every consumer can see which build it loaded
FLAGS += ["-DMUX_EXTRA_FLAGS=\"" + " ".join(EXTRA).replace('"', "") + "\""]
STAMP = SO + ".flags"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stamp_text() -> str:
    return " ".join([NVCC] + FLAGS)


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    # a build with other flags (e.g. an A/B define left in libmux.so) is rebuilt, not reused
    try:
        with open(STAMP) as f:
            if f.read() != _stamp_text():
                return True
    except OSError:
        return True
    t = os.path.getmtime(SO)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "mux.h")]
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    for src in sources():
        obj = os.path.join(HERE, "build", os.path.basename(src) + ".o")
        cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", SO, *objs,
           "-cudart", "static", "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    with open(STAMP, "w") as f:
        f.write(_stamp_text())
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
