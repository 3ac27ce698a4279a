"""Device plumbing: torch owns device memory and streams; the compute is liblramm_cuda."""

from __future__ import annotations

import ctypes
from collections import OrderedDict

import threading

import numpy as np
import torch

from . import _native as N
from .errors import ShapeError

_checked: set[int] = set()


def require_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("liblramm_cuda needs a CUDA device (sm_100a); there is no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
    if dev.index not in _checked:
        with torch.cuda.device(dev):
            N.check(N.LIB.lramm_device_check())
        _checked.add(dev.index)
    return dev


def stream_handle(device=None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


class _Workspace:
    """Grow-only scratch per (device, stream); stream ordering makes reuse safe."""

    def __init__(self):
        self.bufs: dict[tuple[int, int], torch.Tensor] = {}

    def get(self, nbytes: int, device: torch.device) -> torch.Tensor:
        key = (device.index, torch.cuda.current_stream(device).cuda_stream)
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                del self.bufs[key]
                del buf
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            self.bufs[key] = buf
        return buf


WORKSPACE = _Workspace()


def dtype_code(t) -> int:
    if t.dtype in (torch.float32, np.float32):
        return N.F32
    if t.dtype in (torch.float64, np.float64):
        return N.F64
    raise ShapeError(f"unsupported dtype {t.dtype}")


def to_device_matrix(a, device: torch.device, keep_f32: bool = True) -> torch.Tensor:
    """2-D contiguous float32/float64 device tensor (float32 kept: it upcasts exactly on device)."""
    if isinstance(a, torch.Tensor):
        t = a
        if t.dtype not in (torch.float32, torch.float64) or (t.dtype == torch.float32 and not keep_f32):
            t = t.to(torch.float64)
        return t.to(device).contiguous()
    arr = np.asarray(a)
    if arr.dtype != np.float32 or not keep_f32:
        arr = np.asarray(arr, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device)


class OmegaCache:
    """Gaussian test matrices exactly as the reference draws them (rsvd.py:56, matcore.py:89-92):
    generated on the device by lramm_omega (bit-identical to NumPy's Philox + standard_normal,
    tests/test_gpu_omega.py), cached per (seed, ncols, width) on the device and, for the host
    C-ABI path, as a page-locked host copy."""

    def __init__(self, capacity: int = 16):
        self.capacity = capacity
        self.host: OrderedDict = OrderedDict()
        self.dev: OrderedDict = OrderedDict()
        self.lock = threading.RLock()  # host API callers may run on several threads

    @staticmethod
    def philox_key(seed: int, ncols: int, width: int):
        entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF, 0x534B, int(ncols), int(width)]
        key = np.random.Philox(np.random.SeedSequence(entropy)).state["state"]["key"]
        return int(key[0]), int(key[1])

    def _put(self, table, key, value):
        table[key] = value
        if len(table) > self.capacity:
            table.popitem(last=False)

    def device_omega(self, seed: int, ncols: int, width: int, device: torch.device) -> torch.Tensor:
        with self.lock:
            return self._device_omega(seed, ncols, width, device)

    def _device_omega(self, seed: int, ncols: int, width: int, device: torch.device) -> torch.Tensor:
        key = (int(seed), int(ncols), int(width), device.index)
        t = self.dev.get(key)
        if t is None:
            from . import _native as N

            t = torch.empty((ncols, width), dtype=torch.float64, device=device)
            wsz = N.LIB.lramm_omega_ws(ncols, width)
            ws = WORKSPACE.get(wsz, device)
            k0, k1 = self.philox_key(seed, ncols, width)
            N.check(N.LIB.lramm_omega(k0, k1, ncols, width, ptr(t), ptr(ws), wsz, stream_handle(device)))
            if not torch.cuda.is_current_stream_capturing():
                # consumers on other streams (the host C ABI's own streams) read it in place
                torch.cuda.current_stream(device).synchronize()
            self._put(self.dev, key, t)
        else:
            self.dev.move_to_end(key)
        return t

    def host_omega(self, seed: int, ncols: int, width: int) -> np.ndarray:
        with self.lock:
            return self._host_omega(seed, ncols, width)

    def _host_omega(self, seed: int, ncols: int, width: int) -> np.ndarray:
        key = (int(seed), int(ncols), int(width))
        pinned = self.host.get(key)
        if pinned is None:
            dev = require_device()
            pinned = torch.empty((ncols, width), dtype=torch.float64, pin_memory=True)
            pinned.copy_(self.device_omega(seed, ncols, width, dev))
            self._put(self.host, key, pinned)
        else:
            self.host.move_to_end(key)
        return pinned.numpy()


OMEGA = OmegaCache()
