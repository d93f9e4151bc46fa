"""Data-residency helpers: the caller side of the kernels' ``present(f, fn)`` contract.

Mirrors Solomon's intuitive data directives (the reference's
catalog ``pkg/src/pragmaport/data/mappings.reg:74-104,345-347,366-367``) as thin torch
utilities over host numpy arrays:

==========================  =========================================  ==================
Solomon macro               OpenACC lowering (mappings.reg)            here
==========================  =========================================  ==================
MALLOC_ON_DEVICE(a, ...)    acc enter data create(a, ...)              malloc_on_device
FREE_FROM_DEVICE(a, ...)    acc exit data delete(a, ...)               free_from_device
MEMCPY_H2D(a, ...)          acc update device(a, ...)                  memcpy_h2d
MEMCPY_D2H(a, ...)          acc update host(a, ...)                    memcpy_d2h
DATA_ACCESS_BY_DEVICE(...)  acc data ...                               data_access_by_device
DATA_ACCESS_BY_HOST(...)    acc host_data ... (use_device)             data_access_by_host
USE_DEVICE_DATA_FROM_HOST   acc host_data use_device(a, ...)           use_device_data_from_host
(present clause)            present(a)                                 present
SYNCHRONIZE()               acc wait                                   synchronize
==========================  =========================================  ==================

The mapping is keyed by the host array's buffer address, like an OpenACC
present table. Device mirrors are CUDA tensors on the current device; there is
no CPU fallback (``present`` on an unmapped array raises, as an OpenACC runtime
aborts on a missing ``present``).
"""
from __future__ import annotations

import contextlib
import threading

import numpy as np
import torch

from ._lib import SolomonError

_table: dict[int, tuple[np.ndarray, torch.Tensor, int]] = {}  # addr -> (host, device, refcount)
_lock = threading.Lock()


def _key(a: np.ndarray) -> int:
    if not isinstance(a, np.ndarray) or not a.flags.c_contiguous:
        raise SolomonError("residency helpers take C-contiguous numpy arrays")
    return a.__array_interface__["data"][0]


def _require_gpu() -> None:
    if not torch.cuda.is_available():
        raise SolomonError("no CUDA device: data cannot be made device-resident (no CPU fallback)")


def malloc_on_device(*arrays: np.ndarray) -> None:
    """MALLOC_ON_DEVICE: allocate (uninitialised) device mirrors; reference-counted."""
    _require_gpu()
    with _lock:
        for a in arrays:
            k = _key(a)
            if k in _table:
                h, d, rc = _table[k]
                _table[k] = (h, d, rc + 1)
            else:
                d = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device="cuda")
                _table[k] = (a, d, 1)


def free_from_device(*arrays: np.ndarray) -> None:
    """FREE_FROM_DEVICE: drop one reference; the mirror is released at zero."""
    with _lock:
        for a in arrays:
            k = _key(a)
            if k not in _table:
                raise SolomonError("free_from_device: array is not present on the device")
            h, d, rc = _table[k]
            if rc > 1:
                _table[k] = (h, d, rc - 1)
            else:
                del _table[k]


def present(a: np.ndarray) -> torch.Tensor:
    """The device mirror of ``a`` (the ``present`` clause)."""
    with _lock:
        k = _key(a)
        if k not in _table:
            raise SolomonError("present: array is not on the device (missing MALLOC_ON_DEVICE / data region)")
        return _table[k][1]


def is_present(a: np.ndarray) -> bool:
    with _lock:
        return _key(a) in _table


def memcpy_h2d(*arrays: np.ndarray) -> None:
    """MEMCPY_H2D (acc update device): host -> device mirror, stream-ordered."""
    for a in arrays:
        present(a).copy_(torch.from_numpy(a), non_blocking=False)


def memcpy_d2h(*arrays: np.ndarray) -> None:
    """MEMCPY_D2H (acc update host): device mirror -> host, synchronous."""
    for a in arrays:
        np.copyto(a, present(a).cpu().numpy())


def synchronize() -> None:
    """SYNCHRONIZE (acc wait)."""
    torch.cuda.synchronize()


def _refcount(a: np.ndarray) -> int:
    with _lock:
        entry = _table.get(_key(a))
        return entry[2] if entry else 0


@contextlib.contextmanager
def data_access_by_device(copyin=(), copyout=(), copy=(), create=()):
    """DATA_ACCESS_BY_DEVICE: a structured data region (acc data copyin/copyout/copy/create).

    present_or_* semantics, as OpenACC data regions: an array already present (an
    enclosing region or MALLOC_ON_DEVICE) only gains a reference -- copy-in happens
    when its count goes 0 -> 1 and copy-out when it returns 1 -> 0, so a nested
    region neither overwrites newer device data nor copies out early."""
    arrays = list({_key(a): a for a in (*copyin, *copyout, *copy, *create)}.values())  # one reference each
    fresh = [a for a in arrays if _refcount(a) == 0]
    fresh_keys = {_key(a) for a in fresh}
    malloc_on_device(*arrays)
    try:
        memcpy_h2d(*[a for a in (*copyin, *copy) if _key(a) in fresh_keys])
        yield
        memcpy_d2h(*[a for a in (*copyout, *copy) if _refcount(a) == 1])
    finally:
        free_from_device(*arrays)


@contextlib.contextmanager
def data_access_by_host(*arrays: np.ndarray):
    """DATA_ACCESS_BY_HOST / USE_DEVICE_DATA_FROM_HOST (``acc host_data use_device(a, ...)``,
    ``omp target data use_device_ptr(a, ...)``, mappings.reg:345-347,366-367):
    inside the region host code addresses the DEVICE copies of present arrays -- to hand them
    to a library or a drop-in call that takes device pointers. Yields the device tensors in
    argument order (one tensor for one array). Every array must already be present (an
    enclosing DATA_ACCESS_BY_DEVICE or MALLOC_ON_DEVICE), as ``use_device`` requires; the
    region moves no data."""
    mirrors = tuple(present(a) for a in arrays)
    yield mirrors[0] if len(mirrors) == 1 else mirrors


use_device_data_from_host = data_access_by_host
