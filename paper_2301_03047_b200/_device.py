"""Device plumbing for the host layer: numpy <-> CUDA tensors, streams and a
growable workspace pool. PyTorch is used only for device memory, streams and
torch.distributed; every computation is a libglr_b200 kernel."""

from __future__ import annotations

import numpy as np

from . import _native as N


def torch():
    import torch as _t
    return _t


def device():
    N.load(require_gpu=True)
    return torch().device("cuda", torch().cuda.current_device())


def to_dev(a, dtype=None):
    """numpy (or torch) array -> contiguous CUDA tensor."""
    t = torch()
    if isinstance(a, t.Tensor):
        out = a.to(device=device(), dtype=dtype) if dtype is not None else a.to(device())
        return out.contiguous()
    arr = np.ascontiguousarray(a)
    out = t.from_numpy(arr).to(device(), non_blocking=False)
    if dtype is not None:
        out = out.to(dtype)
    return out.contiguous()


def f64(a):
    return to_dev(np.asarray(a, dtype=np.float64))


def i32(a):
    return to_dev(np.asarray(a, dtype=np.int32))


def host(t) -> np.ndarray:
    return t.detach().cpu().numpy()


def host_pinned(t) -> np.ndarray:
    """Device tensor -> numpy array backed by page-locked memory (one DMA at
    full PCIe/C2C rate; torch's pinned-block cache makes the allocation free
    in steady state, and the array keeps its block alive)."""
    out = torch().empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    out.copy_(t.detach())
    return out.numpy()


def empty(shape, dtype):
    return torch().empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    return torch().zeros(shape, dtype=dtype, device=device())


def stream() -> int:
    return N.stream_ptr()


class Workspace:
    """Named scratch buffers that only grow (no allocation in steady state)."""

    def __init__(self):
        self._bufs: dict[str, object] = {}

    def get(self, name: str, nbytes: int):
        t = torch()
        nbytes = max(int(nbytes), 256)
        buf = self._bufs.get(name)
        if buf is None or buf.numel() < nbytes:
            buf = t.empty(nbytes, dtype=t.uint8, device=device())
            self._bufs[name] = buf
        return buf


_WS: Workspace | None = None


def workspace() -> Workspace:
    global _WS
    if _WS is None:
        _WS = Workspace()
    return _WS
