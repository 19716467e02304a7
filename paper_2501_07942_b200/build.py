"""Build the sm_100a product library in-tree (paper_2501_07942_b200/_lib/libttgbf.so).

Five objects, compiled in parallel and linked into one library: api.cu (the
TT step engine; every csrc/*.cuh) once per entry-point group
(-DTTGBF_API_PART=1..4: prior+measurement, time updates, persistent run,
primitives) and dense.cu (the dense grid filter; common.cuh + measure.cuh
only).  Objects are rebuilt only when one of their sources is newer.
"""

from __future__ import annotations

import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIBDIR = os.path.join(HERE, "_lib")
# tuning variants: TTGBF_LIB_VARIANT=tag TTGBF_NVCC_FLAGS="-D..." -> libttgbf_tag.so (loaded by _abi with the same tag)
VARIANT = os.environ.get("TTGBF_LIB_VARIANT", "")
OUT = os.path.join(LIBDIR, "libttgbf%s.so" % ("_" + VARIANT if VARIANT else ""))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
HEADER = os.path.join(ROOT, "include", "ttgbf.h")

FLAGS = [
    "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "--extended-lambda", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]


def _srcs(names):
    return [os.path.join(CSRC, f) for f in names] + [HEADER]


def units():
    cuh = sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))
    api = os.path.join(CSRC, "api.cu")
    out = {f"api{k}": (api, _srcs(["api.cu"] + cuh), [f"-DTTGBF_API_PART={k}"]) for k in (1, 2, 3, 4)}
    out["dense"] = (os.path.join(CSRC, "dense.cu"), _srcs(["dense.cu", "common.cuh", "measure.cuh"]), [])
    return out


def sources():
    out = set()
    for _, deps, _ in units().values():
        out.update(deps)
    return sorted(out)


def _obj(name):
    return os.path.join(LIBDIR, f"{name}{'_' + VARIANT if VARIANT else ''}.o")


def _stale(path, deps):
    return not os.path.exists(path) or os.path.getmtime(path) < max(os.path.getmtime(s) for s in deps)


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    return os.path.getmtime(OUT) >= max(os.path.getmtime(s) for s in sources())


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(LIBDIR, exist_ok=True)
    t0 = time.time()
    procs = {}
    extra = os.environ.get("TTGBF_NVCC_FLAGS", "").split()
    for name, (src, deps, defs) in units().items():
        obj = _obj(name)
        if force or _stale(obj, deps):
            cmd = [NVCC] + FLAGS + defs + extra + ["-c", "-o", obj + ".tmp", src]
            procs[name] = (obj, subprocess.Popen(cmd, cwd=CSRC, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                                 text=True))
    for name, (obj, proc) in procs.items():
        log = proc.communicate()[0]
        if proc.returncode != 0:
            sys.stderr.write(log)
            raise RuntimeError(f"nvcc failed compiling {name}.cu")
        with open(os.path.join(LIBDIR, f"ptxas_{name}{'_' + VARIANT if VARIANT else ''}.log"), "w") as f:
            f.write(log)
        os.replace(obj + ".tmp", obj)
    tmp = OUT + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + [_obj(n) for n in units()]
    proc = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed linking libttgbf.so")
    os.replace(tmp, OUT)
    if verbose:
        print(f"built {OUT} in {time.time() - t0:.0f}s", flush=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
