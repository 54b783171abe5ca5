"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds none of the stencil arithmetic: it only draws numbers.
Both the CPU oracle (tests, bench ``cpu_baseline``) and the CUDA path consume
the arrays produced here, so parity compares the two on identical inputs.

Generator (DESIGN.md §6 "Input recipe"): counter-based splitmix64.  Element
``n`` (0-based, row-major over the whole array, boundary ring included) of
array ``a`` of a workload with seed ``s`` is

    x  = stream_seed(s, a) + (n + 1) * 0x9E3779B97F4A7C15      (mod 2**64)
    z  = splitmix64_mix(x)

and is mapped to
    f32:  (z >> 40) * 2**-24          uniform on [0, 1) with 24 random bits
    f64:  (z >> 11) * 2**-53          uniform on [0, 1) with 53 random bits
    i32:  z >> 63                     Bernoulli(1/2) cell (gameoflife soup)

The value range follows DESIGN.md reading R12 (the paper states none).  The
same generator exists twice: in numpy (host, any size, chunked) and in torch
(device, for the multi-GiB bench grids); a GPU test checks they agree bit for
bit.  Seeds: ``0x230111389 + config_index`` (BASELINE.json configs order).
"""
from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
STREAM = 0xD1B54A32D192ED03
MASK64 = (1 << 64) - 1
BASE_SEED = 0x230111389

_NP_DT = {"f32": np.float32, "f64": np.float64, "i32": np.int32}


def stream_seed(seed: int, array_index: int) -> int:
    """Seed of the ``array_index``-th array of a workload (independent streams)."""
    return (seed ^ ((array_index * STREAM) & MASK64)) & MASK64


def _mix_np(x: np.ndarray) -> np.ndarray:
    x = (x ^ (x >> np.uint64(30))) * np.uint64(M1)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(M2)
    return x ^ (x >> np.uint64(31))


def _map_np(z: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "f32":
        return ((z >> np.uint64(40)).astype(np.float64) * 2.0**-24).astype(np.float32)
    if dtype == "f64":
        return (z >> np.uint64(11)).astype(np.float64) * 2.0**-53
    if dtype == "i32":
        return (z >> np.uint64(63)).astype(np.int32)
    raise ValueError(f"unknown dtype {dtype!r}")


def generate_np(shape, dtype: str, seed: int, array_index: int = 0,
                chunk: int = 1 << 22) -> np.ndarray:
    """Host array of ``shape`` (x fastest = last axis) filled by the recipe."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=_NP_DT[dtype])
    s = np.uint64(stream_seed(seed, array_index))
    with np.errstate(over="ignore"):
        for a in range(0, n, chunk):
            b = min(n, a + chunk)
            ctr = np.arange(a + 1, b + 1, dtype=np.uint64)
            x = s + ctr * np.uint64(GOLDEN)
            out[a:b] = _map_np(_mix_np(x), dtype)
    return out.reshape(shape)


def generate_torch(shape, dtype: str, seed: int, array_index: int = 0,
                   device="cuda", chunk: int = 1 << 26):
    """Same recipe with torch int64 ops (two's-complement wrap = mod 2**64)."""
    import torch

    def s64(v: int) -> int:          # reinterpret a uint64 constant as int64
        v &= MASK64
        return v - (1 << 64) if v >= (1 << 63) else v

    def lsr(x, k: int):              # logical shift right on int64
        return (x >> k) & ((1 << (64 - k)) - 1)

    tdt = {"f32": torch.float32, "f64": torch.float64, "i32": torch.int32}[dtype]
    n = 1
    for d in shape:
        n *= int(d)
    out = torch.empty(n, dtype=tdt, device=device)
    s = s64(stream_seed(seed, array_index))
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        x = torch.arange(a + 1, b + 1, dtype=torch.int64, device=device)
        x = x * s64(GOLDEN) + s
        x = (x ^ lsr(x, 30)) * s64(M1)
        x = (x ^ lsr(x, 27)) * s64(M2)
        z = x ^ lsr(x, 31)
        if dtype == "f32":
            out[a:b] = (lsr(z, 40).to(torch.float64) * 2.0**-24).to(torch.float32)
        elif dtype == "f64":
            out[a:b] = lsr(z, 11).to(torch.float64) * 2.0**-53
        else:
            out[a:b] = lsr(z, 63).to(torch.int32)
        del x, z
    return out.view(*[int(d) for d in shape])
