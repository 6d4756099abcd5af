"""ctypes view of the C oracle (oracle/libkgo.so).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module.
The product package never imports it.  See kgo_aes.h for what is computed
and which FIPS-197 / SP 800-38A passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkgo.so")
ENCRYPT, DECRYPT = 0, 1
MODE_CBC, MODE_ECB = 0, 1

_lib = None


def build() -> str:
    """Compile the oracle (plain C99, no intrinsics) into oracle/libkgo.so."""
    srcs = [os.path.join(_HERE, f) for f in ("kgo_aes.c", "kgo_pages.c")]
    if os.path.exists(LIB_PATH) and all(
            os.path.getmtime(LIB_PATH) >= os.path.getmtime(s) for s in srcs + [os.path.join(_HERE, "kgo_aes.h")]):
        return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-D_POSIX_C_SOURCE=200809L",
                           "-Wall", "-o", tmp] + srcs + ["-lpthread"])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        u8p = ctypes.c_void_p
        L.kgo_init.restype = None
        L.kgo_gf_mul.argtypes = [ctypes.c_uint8, ctypes.c_uint8]
        L.kgo_gf_mul.restype = ctypes.c_uint8
        L.kgo_xtime.argtypes = [ctypes.c_uint8]
        L.kgo_xtime.restype = ctypes.c_uint8
        L.kgo_sbox.argtypes = [ctypes.c_uint8]
        L.kgo_sbox.restype = ctypes.c_uint8
        L.kgo_inv_sbox.argtypes = [ctypes.c_uint8]
        L.kgo_inv_sbox.restype = ctypes.c_uint8
        for name in ("kgo_sub_bytes", "kgo_shift_rows", "kgo_mix_columns",
                     "kgo_inv_sub_bytes", "kgo_inv_shift_rows", "kgo_inv_mix_columns"):
            getattr(L, name).argtypes = [u8p]
            getattr(L, name).restype = None
        L.kgo_add_round_key.argtypes = [u8p, u8p]
        L.kgo_add_round_key.restype = None
        L.kgo_key_expansion.argtypes = [u8p, ctypes.c_int, u8p]
        L.kgo_key_expansion.restype = ctypes.c_int
        L.kgo_cipher.argtypes = [u8p, u8p, u8p, ctypes.c_int]
        L.kgo_cipher.restype = None
        L.kgo_inv_cipher.argtypes = [u8p, u8p, u8p, ctypes.c_int]
        L.kgo_inv_cipher.restype = None
        L.kgo_pages.argtypes = [ctypes.c_int, ctypes.c_int, u8p, ctypes.c_int, u8p, u8p,
                                ctypes.c_uint64, ctypes.c_uint32, u8p, ctypes.c_int]
        L.kgo_pages.restype = ctypes.c_int
        L.kgo_init()
        _lib = L
    return _lib


def _buf(b) -> np.ndarray:
    a = np.frombuffer(bytes(b), dtype=np.uint8) if isinstance(b, (bytes, bytearray)) else np.ascontiguousarray(b, dtype=np.uint8)
    return a


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def gf_mul(a: int, b: int) -> int:
    return lib().kgo_gf_mul(a, b)


def xtime(a: int) -> int:
    return lib().kgo_xtime(a)


def sbox(x: int) -> int:
    return lib().kgo_sbox(x)


def inv_sbox(x: int) -> int:
    return lib().kgo_inv_sbox(x)


def step(name: str, state: bytes) -> bytes:
    """Apply one FIPS-197 round transformation (sub_bytes, shift_rows, ...)."""
    s = np.frombuffer(bytes(state), dtype=np.uint8).copy()
    getattr(lib(), "kgo_" + name)(_ptr(s))
    return s.tobytes()


def add_round_key(state: bytes, rk: bytes) -> bytes:
    s = np.frombuffer(bytes(state), dtype=np.uint8).copy()
    k = np.frombuffer(bytes(rk), dtype=np.uint8).copy()
    lib().kgo_add_round_key(_ptr(s), _ptr(k))
    return s.tobytes()


def key_expansion(key: bytes) -> tuple[int, bytes]:
    k = np.frombuffer(bytes(key), dtype=np.uint8).copy()
    w = np.zeros(240, dtype=np.uint8)
    nr = lib().kgo_key_expansion(_ptr(k), len(key), _ptr(w))
    if nr < 0:
        raise ValueError("bad key length")
    return nr, w[: 16 * (nr + 1)].tobytes()


def cipher(key: bytes, block: bytes) -> bytes:
    nr, w = key_expansion(key)
    wa = np.frombuffer(w, dtype=np.uint8).copy()
    i = np.frombuffer(bytes(block), dtype=np.uint8).copy()
    o = np.zeros(16, dtype=np.uint8)
    lib().kgo_cipher(_ptr(i), _ptr(o), _ptr(wa), nr)
    return o.tobytes()


def inv_cipher(key: bytes, block: bytes) -> bytes:
    nr, w = key_expansion(key)
    wa = np.frombuffer(w, dtype=np.uint8).copy()
    i = np.frombuffer(bytes(block), dtype=np.uint8).copy()
    o = np.zeros(16, dtype=np.uint8)
    lib().kgo_inv_cipher(_ptr(i), _ptr(o), _ptr(wa), nr)
    return o.tobytes()


def pages(direction: int, mode: int, key: bytes, data, n_pages: int, page_bytes: int,
          ivs=None, threads: int = 1, out: np.ndarray | None = None) -> np.ndarray:
    """Per-page CBC (mode 0) / ECB (mode 1) over a flat uint8 buffer; returns uint8 array.
    If out is given (may be `data` itself for in-place), the result is written there."""
    d = _buf(data)
    if d.size != n_pages * page_bytes:
        raise ValueError("data size != n_pages*page_bytes")
    o = np.empty_like(d) if out is None else out
    k = np.frombuffer(bytes(key), dtype=np.uint8).copy()
    iv = None if ivs is None else _buf(ivs)
    rc = lib().kgo_pages(direction, mode, _ptr(k), len(key), _ptr(d), _ptr(o), n_pages, page_bytes,
                         None if iv is None else _ptr(iv), threads)
    if rc != 0:
        raise ValueError("kgo_pages rejected its arguments")
    return o
