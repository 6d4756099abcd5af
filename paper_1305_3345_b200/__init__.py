"""Thin Python binding of the KGPU page-crypto C ABI (include/kg.h).

Argument marshalling only: every step of the hot path runs in
libkgpu.so's CUDA kernels and runtime.  The names mirror the C ABI without
the ``kg_`` prefix.  torch is used only to hand in tensors (device or pinned
host memory) and streams; any other object exposing ``data_ptr()`` or a
raw integer address also works.

There is no CPU fallback: if libkgpu.so is missing, importing this module
raises ImportError (build it with ``make`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KG_LIBKGPU") or os.path.join(_HERE, "libkgpu.so")  # override: experiments only

ENCRYPT, DECRYPT = 0, 1
MODE_CBC, MODE_ECB = 0, 1
OK, EINVAL, ENOKEY, ENOTINIT, EAGAIN, ENOMEM, ECUDA, ENOTSUP, ETICKET = 0, -1, -2, -3, -4, -5, -6, -7, -8
MAX_KEYS = 256
MAX_INFLIGHT = 65536
DEFAULT_STAGING_SLOTS = 6  # kg_set_pipeline's default slot count (include/kg.h)

#: every symbol include/kg.h declares
ABI_SYMBOLS = ("kg_init", "kg_set_key", "kg_submit_pages", "kg_wait", "kg_poll", "kg_shutdown",
               "kg_strerror", "kg_set_pipeline", "kg_launch_count", "kg_set_host_path",
               "kg_nsk_start", "kg_nsk_stop", "kg_nsk_dispatch", "kg_alloc_pinned", "kg_free_pinned",
               "kg_submit_pages_keyed", "kg_dispatch_threshold", "kg_nsk_calibration")
NSK_DIRECT, NSK_NOCAL = 1, 2
HOST_STAGED, HOST_ZEROCOPY, HOST_AUTO = 0, 1, 2

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `make` (or __graft_entry__.build()); "
                      "there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)
_lib.kg_init.argtypes = [ctypes.c_int]
_lib.kg_init.restype = ctypes.c_int
_lib.kg_set_key.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
_lib.kg_set_key.restype = ctypes.c_int
_lib.kg_submit_pages.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                 ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
_lib.kg_submit_pages.restype = ctypes.c_int64
_lib.kg_submit_pages_keyed.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                       ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
_lib.kg_submit_pages_keyed.restype = ctypes.c_int64
_lib.kg_wait.argtypes = [ctypes.c_int64]
_lib.kg_wait.restype = ctypes.c_int
_lib.kg_poll.argtypes = [ctypes.c_int64]
_lib.kg_poll.restype = ctypes.c_int
_lib.kg_shutdown.argtypes = []
_lib.kg_shutdown.restype = ctypes.c_int
_lib.kg_strerror.argtypes = [ctypes.c_int]
_lib.kg_strerror.restype = ctypes.c_char_p
_lib.kg_set_pipeline.argtypes = [ctypes.c_uint64, ctypes.c_int]
_lib.kg_set_pipeline.restype = ctypes.c_int
_lib.kg_set_host_path.argtypes = [ctypes.c_int, ctypes.c_uint64]
_lib.kg_set_host_path.restype = ctypes.c_int
_lib.kg_nsk_start.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint32]
_lib.kg_nsk_start.restype = ctypes.c_int
_lib.kg_nsk_stop.argtypes = []
_lib.kg_nsk_stop.restype = ctypes.c_int
_lib.kg_nsk_dispatch.argtypes = [ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
_lib.kg_nsk_dispatch.restype = ctypes.c_int
_lib.kg_alloc_pinned.argtypes = [ctypes.c_uint64]
_lib.kg_alloc_pinned.restype = ctypes.c_void_p
_lib.kg_free_pinned.argtypes = [ctypes.c_void_p]
_lib.kg_free_pinned.restype = ctypes.c_int


class CalibPoint(ctypes.Structure):
    """kg_calib_point (include/kg.h)."""
    _fields_ = [("bytes", ctypes.c_uint64), ("nsk_us", ctypes.c_double), ("launch_us", ctypes.c_double)]


_lib.kg_dispatch_threshold.argtypes = [ctypes.POINTER(CalibPoint), ctypes.c_int]
_lib.kg_dispatch_threshold.restype = ctypes.c_uint64
_lib.kg_nsk_calibration.argtypes = [ctypes.POINTER(CalibPoint), ctypes.c_int]
_lib.kg_nsk_calibration.restype = ctypes.c_int
_lib.kg_launch_count.argtypes = []
_lib.kg_launch_count.restype = ctypes.c_uint64


class KgError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        self.code = int(code)
        super().__init__(f"{where}: {strerror(code)} ({code})" if where else f"{strerror(code)} ({code})")


def _check(rc: int, where: str) -> int:
    if rc < 0:
        raise KgError(rc, where)
    return rc


def _addr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):  # numpy (must be pinned/registered to be accepted)
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)!r}")


def _stream(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    if hasattr(s, "cuda_stream"):
        return s.cuda_stream
    raise TypeError(f"not a stream: {type(s)!r}")


def strerror(code: int) -> str:
    return _lib.kg_strerror(int(code)).decode()


def init(device: int = 0) -> None:
    _check(_lib.kg_init(int(device)), "kg_init")


def set_key(key_id: int, key: bytes) -> None:
    key = bytes(key)
    _check(_lib.kg_set_key(int(key_id), key, len(key)), "kg_set_key")


def submit_pages(direction: int, mode: int, inp, out, n_pages: int, page_bytes: int, ivs, key_id: int,
                 stream=None) -> int:
    """Enqueue one batch; returns the ticket (raises KgError on a negative status)."""
    rc = _lib.kg_submit_pages(int(direction), int(mode), _addr(inp), _addr(out), int(n_pages), int(page_bytes),
                              _addr(ivs), int(key_id), _stream(stream))
    return _check(rc, "kg_submit_pages")


def submit_pages_raw(direction, mode, inp, out, n_pages, page_bytes, ivs, key_id, stream=None) -> int:
    """Like submit_pages but returns the raw status/ticket without raising."""
    return _lib.kg_submit_pages(int(direction), int(mode), _addr(inp), _addr(out), int(n_pages), int(page_bytes),
                                _addr(ivs), int(key_id), _stream(stream))


def submit_pages_keyed(direction: int, mode: int, inp, out, n_pages: int, page_bytes: int, ivs, key_ids,
                       key_bytes: int, stream=None) -> int:
    """Mixed-key batch: page p under key key_ids[p] (uint16 tensor); returns the ticket."""
    rc = _lib.kg_submit_pages_keyed(int(direction), int(mode), _addr(inp), _addr(out), int(n_pages), int(page_bytes),
                                    _addr(ivs), _addr(key_ids), int(key_bytes), _stream(stream))
    return _check(rc, "kg_submit_pages_keyed")


def wait(ticket: int) -> None:
    _check(_lib.kg_wait(int(ticket)), "kg_wait")


def wait_raw(ticket: int) -> int:
    return _lib.kg_wait(int(ticket))


def poll(ticket: int) -> bool:
    return bool(_check(_lib.kg_poll(int(ticket)), "kg_poll"))


def poll_raw(ticket: int) -> int:
    return _lib.kg_poll(int(ticket))


def shutdown() -> None:
    _check(_lib.kg_shutdown(), "kg_shutdown")


def set_pipeline(chunk_bytes: int, slots: int) -> None:
    _check(_lib.kg_set_pipeline(int(chunk_bytes), int(slots)), "kg_set_pipeline")


def set_host_path(mode: int, zc_max_bytes: int = 1 << 20) -> None:
    _check(_lib.kg_set_host_path(int(mode), int(zc_max_bytes)), "kg_set_host_path")


def nsk_start(ctas: int = 0, flags: int = 0, idle_ms: int = 0) -> None:
    """Start the Non-Stop Kernel (persistent service kernel, row f3)."""
    _check(_lib.kg_nsk_start(int(ctas), int(flags), int(idle_ms)), "kg_nsk_start")


def nsk_stop() -> None:
    _check(_lib.kg_nsk_stop(), "kg_nsk_stop")


def nsk_dispatch(max_bytes: int = 0) -> int:
    """Route requests <= max_bytes to the NSK, larger ones to launches (0 = calibrate).
    Returns the threshold in use."""
    out = ctypes.c_uint64(0)
    _check(_lib.kg_nsk_dispatch(int(max_bytes), ctypes.byref(out)), "kg_nsk_dispatch")
    return int(out.value)


def dispatch_threshold(points) -> int:
    """kg_dispatch_threshold over [(bytes, nsk_us, launch_us), ...]."""
    arr = (CalibPoint * max(1, len(points)))(*[CalibPoint(int(b), float(n), float(l)) for b, n, l in points])
    return int(_lib.kg_dispatch_threshold(arr, len(points)))


def nsk_calibration():
    """The last calibration's samples [(bytes, nsk_us, launch_us), ...]."""
    arr = (CalibPoint * 16)()
    n = _check(_lib.kg_nsk_calibration(arr, 16), "kg_nsk_calibration")
    return [(int(p.bytes), float(p.nsk_us), float(p.launch_us)) for p in arr[:min(n, 16)]]


def alloc_pinned(nbytes: int):
    """NUMA-local pinned+mapped host buffer as a torch uint8 tensor (freed with free_pinned)."""
    import torch
    p = _lib.kg_alloc_pinned(int(nbytes))
    if not p:
        raise KgError(ENOMEM, "kg_alloc_pinned")
    buf = (ctypes.c_uint8 * int(nbytes)).from_address(p)
    t = torch.frombuffer(buf, dtype=torch.uint8)
    t._kg_base = p  # noqa: SLF001  (keeps the base address for free_pinned)
    return t


def free_pinned(t) -> None:
    base = getattr(t, "_kg_base", None)
    _check(_lib.kg_free_pinned(base if base is not None else _addr(t)), "kg_free_pinned")


def launch_count() -> int:
    return int(_lib.kg_launch_count())


def crypt_pages(direction: int, mode: int, inp, out, n_pages: int, page_bytes: int, ivs, key_id: int,
                stream=None) -> None:
    """submit_pages + wait."""
    wait(submit_pages(direction, mode, inp, out, n_pages, page_bytes, ivs, key_id, stream))


def raw_lib():
    return _lib
