"""TEST-ONLY single-thread emulation of the CUDA step engine.

The engine sources (paper_2501_07942_b200/csrc/*.cuh + api.cu) are written
as CTA-cooperative C++; compiled with g++ -DENGINE_HOSTSIM they run with a
one-thread "CTA" on the CPU.  The CPU suite uses this to check the engine's
decision logic (cross, rounding, stages) and the Python driver against the
oracle without a GPU.  The product package never builds or loads it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2501_07942_b200", "csrc")
OUT = os.path.join(ROOT, "tests", "_build", "libttgbf_hostsim.so")


def build() -> str:
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "ttgbf.h")]
    newest = max(os.path.getmtime(s) for s in srcs)
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-x", "c++", "-DENGINE_HOSTSIM",
           "-o", OUT + ".tmp", os.path.join(CSRC, "api.cu")]
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


class HostBuffer:
    __slots__ = ("a", "nbytes")

    def __init__(self, nbytes):
        self.nbytes = max(int(nbytes), 8)
        self.a = np.zeros(self.nbytes, dtype=np.uint8)

    @property
    def ptr(self) -> int:
        return self.a.ctypes.data


class HostBackend:
    """Same interface as CudaBackend; buffers are host arrays."""

    name = "hostsim"

    def __init__(self):
        from paper_2501_07942_b200 import _abi
        import torch
        self.lib = _abi.bind(ctypes.CDLL(build()), dense=False)
        self.stream_ptr = None
        self.torch = torch
        self.device = torch.device("cpu")

    def empty(self, nbytes):
        return HostBuffer(nbytes)

    def upload(self, arr):
        raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        b = HostBuffer(raw.nbytes)
        b.a[: raw.nbytes] = raw
        return b

    def upload_into(self, buf, arr):
        raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        buf.a[: raw.nbytes] = raw

    def download(self, buf, dtype, count, offset_bytes=0):
        dtype = np.dtype(dtype)
        nb = dtype.itemsize * int(count)
        return buf.a[offset_bytes: offset_bytes + nb].copy().view(dtype)[:count].copy()

    def zero(self, buf):
        buf.a[:] = 0

    def sync(self):
        pass

    def check(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"{what}: rc={rc}")
