"""Seeded synthetic input generators shared by the CUDA path's tests/bench and
the oracle's tests.  This module holds none of the method's arithmetic: it
only draws initial states (the recipe is in DESIGN.md "Input recipe").

The counter-based key() here is the same SplitMix64-based generator that the
oracle (C) and the CUDA kernels each implement on their own (reading R-RNG);
it is used here only to draw initial Wa-Tor grids.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
PH_INIT, PH_FISH_REQ, PH_FISH_DEC, PH_SHARK_REQ, PH_SHARK_DEC, PH_MB_FIELD = range(6)


def sm(x):
    """SplitMix64 output function, vectorised over uint64 arrays."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def key(seed, step, phase, idx):
    """key(seed, step, phase, idx) = sm(sm(sm(seed) ^ step) ^ (phase << 40 | idx))."""
    s = sm(np.uint64(seed)) ^ np.uint64(step)
    return sm(sm(s) ^ ((np.uint64(phase) << np.uint64(40)) | np.asarray(idx, dtype=np.uint64)))


# ------------------------------------------------------------------ microbench
MB_NF = (3, 3, 4, 6)       # fields of thread t's object, [A, A, B, C][t & 3]


def mb_fields(seed: int, t0: int, n: int, chunk: int = 1 << 20) -> np.ndarray:
    """Field values of threads t0 .. t0+n-1 of the microbench (t0 % 4 == 0,
    n % 4 == 0), packed per 4 threads as 16 u32 {A: 3, A: 3, B: 4, C: 6}:
    field k of thread t = low32(key(seed, 0, MB_FIELD, 16 t + k)) (DESIGN.md
    "Input recipe").  Host-resident inputs for the end-to-end bench."""
    assert t0 % 4 == 0 and n % 4 == 0
    out = np.empty(4 * n, dtype=np.uint32)
    # (thread offset within the group of 4, field k) for the 16 packed slots
    toff = np.array([0] * 3 + [1] * 3 + [2] * 4 + [3] * 6, dtype=np.uint64)
    kk = np.array([0, 1, 2, 0, 1, 2, 0, 1, 2, 3, 0, 1, 2, 3, 4, 5], dtype=np.uint64)
    def fill(g0):
        g = np.arange(g0, min(n // 4, g0 + chunk), dtype=np.uint64)
        t = np.uint64(t0) + np.uint64(4) * g[:, None] + toff[None, :]
        out[16 * g0:16 * (g0 + len(g))] = (key(seed, 0, PH_MB_FIELD, np.uint64(16) * t + kk[None, :])
                                           & np.uint64(0xFFFFFFFF)).astype(np.uint32).ravel()
    import concurrent.futures as cf
    import os
    with cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:   # numpy releases the GIL
        list(ex.map(fill, range(0, n // 4, chunk)))
    return out


# ------------------------------------------------------------------ Game of Life
def gol_soup(W: int, H: int, p: float, seed: int) -> np.ndarray:
    """Bernoulli(p) alive bitmap, (H, W) uint8 (BASELINE configs[0]/[3])."""
    rng = np.random.default_rng(seed)
    return (rng.random((H, W)) < p).astype(np.uint8)


PATTERNS = {
    "glider": [(1, 2), (2, 3), (3, 1), (3, 2), (3, 3)],      # (row, col)
    "blinker": [(10, 10), (10, 11), (10, 12)],
    "block": [(5, 5), (5, 6), (6, 5), (6, 6)],
    "beehive": [(5, 6), (5, 7), (6, 5), (6, 8), (7, 6), (7, 7)],
}


def gol_pattern(name: str, W: int = 64, H: int = 64) -> np.ndarray:
    a = np.zeros((H, W), dtype=np.uint8)
    for r, c in PATTERNS[name]:
        a[r % H, c % W] = 1
    return a


# ------------------------------------------------------------------ Wa-Tor
def wator_init(W: int, H: int, seed: int = 42, FB: int = 6, SB: int = 12, SS: int = 6,
               fish_permille: int = 300, shark_permille: int = 50):
    """Per cell c: u = key(seed,0,INIT,c) % 1000; u < 300 -> fish (egg = key % FB);
    u < 350 -> shark (egg = key % SB, energy = SS); else empty."""
    c = np.arange(W * H, dtype=np.uint64)
    k = key(seed, 0, PH_INIT, c)
    u = k % np.uint64(1000)
    kind = np.zeros(W * H, dtype=np.uint8)
    egg = np.zeros(W * H, dtype=np.uint32)
    energy = np.zeros(W * H, dtype=np.uint32)
    fish = u < fish_permille
    shark = (~fish) & (u < fish_permille + shark_permille)
    kind[fish] = 1
    kind[shark] = 2
    egg[fish] = (k[fish] % np.uint64(FB)).astype(np.uint32)
    egg[shark] = (k[shark] % np.uint64(SB)).astype(np.uint32)
    energy[shark] = SS
    return kind.reshape(H, W), egg.reshape(H, W), energy.reshape(H, W)


# ------------------------------------------------------------------ N-body
def nbody_init(n: int, seed: int = 7):
    """x, y in [-1, 1) on a 2^-23 grid, v = 0, m in [1, 2) (fp32-exact values)."""
    rng = np.random.default_rng(seed)
    x = ((rng.integers(0, 1 << 24, n) - (1 << 23)) / float(1 << 23)).astype(np.float32)
    y = ((rng.integers(0, 1 << 24, n) - (1 << 23)) / float(1 << 23)).astype(np.float32)
    m = (1.0 + rng.integers(0, 1 << 23, n) / float(1 << 23)).astype(np.float32)
    z = np.zeros(n, dtype=np.float32)
    return {"x": x, "y": y, "vx": z.copy(), "vy": z.copy(), "m": m, "alive": np.ones(n, dtype=np.uint8)}


# N-body constants (calibrated, then frozen)
NBODY_PARAMS = {"G": 1e-12, "dt": 0.5, "eps": 2.5e-4, "R": 1e-3}


# ------------------------------------------------------------------ microbench
MB_TYPES = [[4, 4, 4], [4, 4, 4, 4], [4, 4, 4, 4, 4, 4]]   # A, B, C (12/16/24 B)
