"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds NO AES/CBC arithmetic: only a counter-based generator
(splitmix64) and the page-range shard arithmetic.  It is the one module
both the oracle-side tests and the CUDA-side callers import (DESIGN.md
"Input recipe").

Generator: 64-bit word i of stream `seed` is splitmix64's finaliser applied
to seed + (i+1)*0x9E3779B97F4A7C15, stored little-endian at byte 8i.

Workload structure: independent pages of
uniformly random bytes (4 KiB in every BASELINE.json config), one uniformly
random 16-byte IV per page, a uniformly random 16/24/32-byte key.  The paper
sizes pages at 4 KiB ("8KB ... is two memory pages").
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

DATA_SEED = 0x4B475055  # "KGPU"
KEY_SEED = DATA_SEED + 1
IV_SEED = DATA_SEED + 2

#: BASELINE.json configs as concrete shapes (n_pages, page_bytes, key_bytes, dir)
PAGE_BYTES = 4096


def splitmix64_words(seed: int, n_words: int, first_word: int = 0) -> np.ndarray:
    """Words first_word .. first_word+n_words-1 of the stream (uint64)."""
    with np.errstate(over="ignore"):
        i = np.arange(first_word + 1, first_word + n_words + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def stream_bytes(seed: int, n_bytes: int, offset: int = 0) -> np.ndarray:
    """n_bytes of the stream starting at byte `offset` (offset % 8 == 0)."""
    if offset % 8:
        raise ValueError("offset must be a multiple of 8")
    n_words = (n_bytes + 7) // 8
    w = splitmix64_words(seed, n_words, offset // 8)
    return w.astype("<u8").view(np.uint8)[:n_bytes].copy()


def make_key(key_bytes: int, seed: int = KEY_SEED) -> bytes:
    return stream_bytes(seed, key_bytes).tobytes()


def make_pages(n_pages: int, page_bytes: int = PAGE_BYTES, seed: int = DATA_SEED,
               first_page: int = 0) -> np.ndarray:
    """Pages [first_page, first_page+n_pages) of the seeded page stream, flat uint8."""
    return stream_bytes(seed, n_pages * page_bytes, first_page * page_bytes)


def make_ivs(n_pages: int, seed: int = IV_SEED, first_page: int = 0) -> np.ndarray:
    return stream_bytes(seed, 16 * n_pages, 16 * first_page)


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous page range [lo, hi) of rank `rank` out of `world`:
    [floor(r*N/W), floor((r+1)*N/W))."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world
