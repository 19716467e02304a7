"""Build the sm_100a product library in-tree (paper_2501_07942_b200/_lib/libttgbf.so)."""

from __future__ import annotations

import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "_lib", "libttgbf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "--extended-lambda", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def sources():
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))]
    return srcs + [os.path.join(ROOT, "include", "ttgbf.h")]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    return os.path.getmtime(OUT) >= max(os.path.getmtime(s) for s in sources())


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp"
    cmd = [NVCC] + FLAGS + ["-o", tmp, os.path.join(CSRC, "api.cu")]
    t0 = time.time()
    proc = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed building libttgbf.so")
    with open(os.path.join(os.path.dirname(OUT), "ptxas.log"), "w") as f:
        f.write(proc.stdout + proc.stderr)
    os.replace(tmp, OUT)
    if verbose:
        print(f"built {OUT} in {time.time() - t0:.0f}s", flush=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
