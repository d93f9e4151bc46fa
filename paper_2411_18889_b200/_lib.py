"""ctypes binding of ``lib/libsolomon_b200.so`` (the sm_100a C-ABI, include/solomon_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute call raises. ``load()`` is the single entry point.
"""
from __future__ import annotations

import ctypes
import pathlib
import threading

import torch

PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libsolomon_b200.so"

# include/solomon_b200.h
B2_OK = 0
B2_EINVAL = -1
B2_EALIGN = -2
B2_ESPACE = -3
B2_ENOMEM = -4
B2_ETIMEOUT = -5
B2_ENOTSUP = -6
B2_POTENTIAL = 1
B2_EXACT = 2
B2_INIT_ACC = 4
B2_KDK_REDUCE = 1
B2_KDK_KICK_END = 2
B2_KDK_KICK_DRIFT = 4

_i, _f, _p, _sz = ctypes.c_int, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t

# name -> (restype, argtypes); every symbol include/solomon_b200.h declares.
SIGNATURES = {
    "calc_acc": (None, [_i, _p, _p, _i, _p, _f]),
    "calc_acc_potential": (None, [_i, _p, _p, _i, _p, _f]),
    "calc_acc_exact": (None, [_i, _p, _p, _i, _p, _f]),
    "calc_acc_potential_exact": (None, [_i, _p, _p, _i, _p, _f]),
    "diffusion3d": (None, [_i, _i, _i, _f, _f, _f, _f, _f, _p, _p]),
    "b2_last_error": (_i, []),
    "b2_error_string": (ctypes.c_char_p, [_i]),
    "b2_version": (ctypes.c_char_p, []),
    "b2_set_poll_timeout_ms": (_i, [ctypes.c_longlong]),
    "b2_poll_timeout_ms": (ctypes.c_longlong, []),
    "b2_fault_status": (_i, [_p, _i, ctypes.POINTER(_i)]),
    "b2_fault_kernel": (ctypes.c_char_p, [_i]),
    "b2_calc_acc_nchunks": (_i, [_i, _i]),
    "b2_calc_acc_workspace_bytes": (_sz, [_i, _i, _i]),
    "b2_calc_acc": (_i, [_i, _p, _p, _i, _p, _f, _i, _p, _sz, _p]),
    "b2_calc_acc_partials": (_i, [_i, _p, _i, _p, _f, _i, _p, _p]),
    "b2_kdk_update": (_i, [_i, _p, _p, _p, _p, _i, _f, _f, _f, _i, _p]),
    "b2_kdk_update_publish": (_i, [_i, _p, _p, _p, _p, _p, _i, _f, _f, _f, _i, _p, _i, _p]),
    "b2_kdk_update_multicast": (_i, [_i, _p, _p, _p, _p, _p, _i, _f, _f, _f, _i, _p]),
    "b2_leapfrog": (_i, [_i, _p, _p, _p, _f, _f, _i, _i, _p, _sz, _p]),
    "b2_leapfrog_workspace_bytes": (_sz, [_i, _i]),
    "b2_diffusion3d": (_i, [_i, _i, _i, _f, _f, _f, _f, _f, _p, _p, _p]),
    "b2_diffusion3d_plan": (_i, [_i, _i, _i, _f, _f, _f, _f, _f, _p, _p, _i, _p]),
    "b2_diffusion3d_slab": (_i, [_i, _i, _i, _f, _f, _f, _f, _f, _p, _p, _p, _p, _i, _i, _p]),
    "b2_diffusion3d_run": (_i, [_i, _i, _i, _f, _f, _f, _f, _f, _p, _p, _i, ctypes.POINTER(_i), _p]),
    "b2_debug_withhold_publish": (_i, [_i]),
    "b2_diffusion3d_run2_planes": (_i, [_i, _i, _i, _f, _f, _f, _f, _f, _p, _p, _i, _i, _i, _i, _p]),
    "b2_diffusion3d_mailbox_bytes": (_sz, [_i, _i]),
    "b2_diffusion3d_slab_edges": (_i, [_i, _i, _i, _f, _f, _f, _f, _f, _p, _p, _p, _p, _p, _p, _i, _i, _p]),
    "b2_diffusion3d_mailbox2_bytes": (_sz, [_i, _i]),
    "b2_diffusion3d_slab_halo2": (_i, [_i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _i, _i, _p]),
    "b2_ipc_handle_bytes": (_sz, []),
    "b2_ipc_export": (_i, [_p, _p, ctypes.POINTER(_sz)]),
    "b2_mc_supported": (_i, [_i]),
    "b2_mc_handle_bytes": (_sz, []),
    "b2_mc_granular_bytes": (_i, [_sz, _i, ctypes.POINTER(_sz)]),
    "b2_mc_create": (_i, [_sz, _i, _i, _p, ctypes.POINTER(_p)]),
    "b2_mc_add_device": (_i, [_p, _i, ctypes.POINTER(_p)]),
    "b2_mc_bind": (_i, [_p, _sz, ctypes.POINTER(_p), ctypes.POINTER(_p)]),
    "b2_mc_release": (_i, [_p]),
    "b2_ipc_import": (_i, [_p, _sz, ctypes.POINTER(_p)]),
    "b2_ipc_close": (_i, [_p, _sz]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


class SolomonError(RuntimeError):
    """A b2_* call returned a non-zero status."""


def load(path: pathlib.Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the C-ABI library. Raises if it is missing."""
    global _lib
    if _lib is not None and path is None:  # fast path: no lock once loaded
        return _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = pathlib.Path(path) if path else LIB_PATH
        if not p.exists():
            raise SolomonError(
                f"{p} not found: build it with `python -m paper_2411_18889_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != B2_OK:
        msg = load().b2_error_string(rc).decode()
        raise SolomonError(f"{what}: {msg} (code {rc})")


def check_fault(device: torch.device | None = None, what: str = "run") -> None:
    """Synchronise ``device``'s current stream and raise if a device-side wait gave up.

    The polling kernels (persistent small-N leapfrog, resident diffusion, the p2p slab
    halo) never hang or trap: a word that does not arrive within the poll timeout
    (``set_poll_timeout``) makes them record a fault and exit. This turns that record
    into a ``SolomonError`` (and clears it, so the device is usable again)."""
    lib = load()
    which = ctypes.c_int(0)
    with on_device(device if device is not None else torch.device("cuda", torch.cuda.current_device())):
        rc = lib.b2_fault_status(stream_handle(device), 1, ctypes.byref(which))
    if rc == B2_ETIMEOUT:
        raise SolomonError(f"{what}: a device-side wait timed out after {lib.b2_poll_timeout_ms() / 1e3:g} s in "
                           f"{lib.b2_fault_kernel(which.value).decode()}; results of that launch are undefined")
    check(rc, what)


def set_poll_timeout(seconds: float) -> None:
    """How long a kernel waits in the GPU for another CTA's / GPU's data before giving up
    (default ``SOLOMON_POLL_TIMEOUT_S`` or 120 s). Applies to later launches."""
    check(load().b2_set_poll_timeout_ms(max(1, int(round(seconds * 1e3)))), "set_poll_timeout")


def require_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise SolomonError(f"{name} must be a CUDA tensor (no CPU fallback); got device {t.device}")


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(device: torch.device | None = None) -> int:
    """cudaStream_t of torch's current stream on ``device`` (cheap path when available)."""
    if _raw_stream is not None:
        idx = device.index if isinstance(device, torch.device) and device.index is not None else \
            torch.cuda.current_device()
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


class on_device:
    """``torch.cuda.device(t.device)`` only when it differs from the current device."""

    __slots__ = ("idx", "prev")

    def __init__(self, device: torch.device):
        self.idx = device.index if device.index is not None else torch.cuda.current_device()
        self.prev = None

    def __enter__(self):
        cur = torch.cuda.current_device()
        if cur != self.idx:
            self.prev = cur
            torch.cuda.set_device(self.idx)
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            torch.cuda.set_device(self.prev)
        return False
