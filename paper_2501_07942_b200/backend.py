"""Device plumbing for the C-ABI: buffers, copies and the stream (PyTorch).

PyTorch is used only to own device memory and the CUDA stream; every
computation runs in the hand-written kernels of ``libttgbf.so``.  The
:class:`CudaBackend` is the only backend the product package provides.
"""

from __future__ import annotations

import numpy as np

from paper_2501_07942_b200 import _abi


class DeviceBuffer:
    __slots__ = ("t", "nbytes")

    def __init__(self, t, nbytes):
        self.t = t
        self.nbytes = nbytes

    @property
    def ptr(self) -> int:
        return int(self.t.data_ptr())


class CudaBackend:
    """Owns the library handle, a device and a stream."""

    name = "cuda"

    def __init__(self, device: int | None = None):
        import torch
        self.lib = _abi.load_library()
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = torch.cuda.current_stream(self.device)
        self.nvtx = torch.cuda.nvtx

    @property
    def stream_ptr(self) -> int:
        return int(self.stream.cuda_stream)

    def empty(self, nbytes: int) -> DeviceBuffer:
        n = max(int(nbytes), 8)
        return DeviceBuffer(self.torch.empty(n, dtype=self.torch.uint8, device=self.device), n)

    def upload(self, arr: np.ndarray) -> DeviceBuffer:
        a = np.ascontiguousarray(arr)
        raw = a.view(np.uint8).reshape(-1)
        buf = self.empty(raw.nbytes)
        if raw.nbytes:
            src = self.torch.from_numpy(raw)
            buf.t[: raw.nbytes].copy_(src, non_blocking=False)
        return buf

    def upload_into(self, buf: DeviceBuffer, arr: np.ndarray) -> None:
        raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        if raw.nbytes:
            buf.t[: raw.nbytes].copy_(self.torch.from_numpy(raw), non_blocking=False)

    def download(self, buf: DeviceBuffer, dtype, count: int, offset_bytes: int = 0) -> np.ndarray:
        dtype = np.dtype(dtype)
        nb = dtype.itemsize * int(count)
        host = buf.t[offset_bytes: offset_bytes + nb].cpu().numpy()
        return host.view(dtype)[:count].copy()

    def zero(self, buf: DeviceBuffer) -> None:
        buf.t.zero_()

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)

    def sync(self) -> None:
        self.torch.cuda.synchronize(self.device)

    def check(self, rc: int, what: str) -> None:
        if rc != 0:
            raise RuntimeError(f"{what}: launch failed ({_abi.status_text(rc)})")
