"""Counter-based seeded input heaps (SURVEY.md §8(d) seeds).

Every value is a pure function of (config, array, instance, index):

    s     = splitmix64(0x13083203 ^ (cfg << 48) ^ (array << 40) ^ instance)
    x[i]  = splitmix64(s + i)            (low 32 bits, as int32)

so any instance can be regenerated alone (oracle samples, multi-GPU shards)
without transfer.  No method arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

SEED = 0x13083203
_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def stream(cfg: int, array: int, instance: int, n: int) -> np.ndarray:
    """n raw 64-bit draws of the (cfg, array, instance) stream."""
    s = splitmix64(np.uint64((SEED ^ (cfg << 48) ^ (array << 40) ^ instance) & 0xFFFFFFFFFFFFFFFF))
    with np.errstate(over="ignore"):
        return splitmix64(s + np.arange(n, dtype=np.uint64))


def uniform_i32(cfg: int, array: int, instance: int, n: int) -> np.ndarray:
    return (stream(cfg, array, instance, n) & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)


# --- per-config input recipes (instances [i0, i1)) ----------------------------

def cfg1_inputs(n: int = 8) -> list[np.ndarray]:
    """Config 1 (App. A.1): A[i]=i+1, B[i]=10(i+1), R[i]=100+i; one instance."""
    i = np.arange(n, dtype=np.int32)
    return [(i + 1)[None, :], (10 * (i + 1))[None, :], (100 + i)[None, :]]


def cfg2_inputs(i0: int, i1: int, n: int = 256) -> list[np.ndarray]:
    """Config 2: A int32[1] random; B int32[n]: constant-filled (a random
    constant) on even instances, random bits {0,1} on odd instances."""
    A = np.stack([uniform_i32(2, 0, i, 1) for i in range(i0, i1)]) if i1 > i0 else np.zeros((0, 1), np.int32)
    rows = []
    for i in range(i0, i1):
        if i % 2 == 0:
            rows.append(np.full(n, uniform_i32(2, 1, i, 1)[0], dtype=np.int32))
        else:
            rows.append((stream(2, 1, i, n) & np.uint64(1)).astype(np.int32))
    B = np.stack(rows) if rows else np.zeros((0, n), np.int32)
    return [A, B]


def cfg3_inputs(i0: int, i1: int, n: int = 1024) -> list[np.ndarray]:
    """Config 3: A int32[n] uniform."""
    return [np.stack([uniform_i32(3, 0, i, n) for i in range(i0, i1)]) if i1 > i0
            else np.zeros((0, n), np.int32)]


def cfg4_inputs(i0: int, i1: int, n: int = 65536, halo: int = 4) -> list[np.ndarray]:
    """Config 4: X0..X2 uniform int32[n+2K]; X3 index array, X3[c] = c except
    with probability 2^-12 where X3[c] = c-1 or c+1."""
    size = n + 2 * halo
    out = []
    for a in range(3):
        out.append(np.stack([uniform_i32(4, a, i, size) for i in range(i0, i1)]) if i1 > i0
                   else np.zeros((0, size), np.int32))
    rows = []
    c = np.arange(size, dtype=np.int64)
    for i in range(i0, i1):
        u = stream(4, 3, i, size)
        hit = (u >> np.uint64(52)) == 0
        step = np.where((u & np.uint64(1)) == 1, 1, -1)
        rows.append(np.where(hit, c + step, c).astype(np.int32))
    out.append(np.stack(rows) if rows else np.zeros((0, size), np.int32))
    return out


def cfg5_inputs(i0: int, i1: int, n: int = 1 << 20) -> list[np.ndarray]:
    """Config 5: A int32[n+2] uniform (halos A[0], A[n+1] never written), B zeros."""
    size = n + 2
    A = np.stack([uniform_i32(5, 0, i, size) for i in range(i0, i1)]) if i1 > i0 else np.zeros((0, size), np.int32)
    return [A, np.zeros((i1 - i0, size), dtype=np.int32)]


def tiny_inputs(rng: np.random.Generator, n_arrays: int, size: int, lo: int = 0, hi: int = 3) -> list[np.ndarray]:
    return [rng.integers(lo, hi, size=(1, size)).astype(np.int32) for _ in range(n_arrays)]
