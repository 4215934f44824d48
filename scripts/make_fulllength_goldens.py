"""Write the full-length BASELINE goldens (oracle only, so the default -m gpu
suite can check the full runs without minutes of CPU work per test):

* tests/golden/gol16384_1000gen_windows.npz -- configs[3]: Game of Life
  16384^2 (p = 0.25, seed 42), 1000 generations.  Three 96 x 96 windows at
  seeded positions; each is the oracle's dense Life (oracle.life_dense) run
  for 1000 generations on the window's light cone -- the initial
  (96 + 2000)^2 region around it -- of which the inner 96 x 96 cells are exact
  (a wrap error of the region travels one cell per generation).
* tests/golden/wator2048_500steps.npz -- configs[1]: Wa-Tor 2048^2 (seed 42,
  FB 6 SB 12 SS 6), the object oracle's (oracle.wator_run) per-step counters
  for 500 steps and the SHA-256 of the final state (kind u8, egg u32, energy
  u32 arrays, C order, little-endian) -- the full arrays would be 3.4 MB.

Calls only oracle/ and the seeded input generator (paper_1810_11765_b200/inputs.py,
which holds none of the method's arithmetic).  ~10 min on one core per part:
    python scripts/make_fulllength_goldens.py [gol] [wator]"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O                      # noqa: E402
from paper_1810_11765_b200 import inputs as I       # noqa: E402

GOL_W = GOL_H = 16384
GOL_G, GOL_WIN, GOL_NWIN, GOL_WSEED = 1000, 96, 3, 1
WT = dict(FB=6, SB=12, SS=6, seed=42)
WT_N, WT_STEPS = 2048, 500


def gol_windows():
    """Window origins (y, x): numpy PCG64 seed 1, the same draws the test makes."""
    rng = np.random.default_rng(GOL_WSEED)
    return [(int(rng.integers(0, GOL_H)), int(rng.integers(0, GOL_W))) for _ in range(GOL_NWIN)]


def make_gol():
    a0 = I.gol_soup(GOL_W, GOL_H, 0.25, 42)
    G, w = GOL_G, GOL_WIN
    wins, outs = gol_windows(), []
    for y, x in wins:
        ys = np.arange(y - G, y + w + G) % GOL_H
        xs = np.arange(x - G, x + w + G) % GOL_W
        region = np.ascontiguousarray(a0[np.ix_(ys, xs)])
        outs.append(O.life_dense(region, G)[G:G + w, G:G + w].astype(np.uint8))
    out = ROOT / "tests" / "golden" / "gol16384_1000gen_windows.npz"
    np.savez_compressed(out, windows=np.array(wins, np.int64), alive=np.stack(outs),
                        meta=np.array([GOL_W, GOL_H, 42, GOL_G, w]), p=np.array([0.25]))
    return out


def state_digest(x, dtype):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.dtype(dtype).newbyteorder("<")).tobytes()).hexdigest()


def make_wator():
    kind, egg, en = I.wator_init(WT_N, WT_N, seed=42)
    k, e, n, c = O.wator_run(kind, egg, en, steps=WT_STEPS, **WT)
    out = ROOT / "tests" / "golden" / "wator2048_500steps.npz"
    np.savez_compressed(out, counters=np.asarray(c, np.int64), kind=k, egg=e, energy=n,
                        meta=np.array([WT_N, WT_N, WT["seed"], WT_STEPS, WT["FB"], WT["SB"], WT["SS"]]))
    return out


if __name__ == "__main__":
    O.build()
    parts = sys.argv[1:] or ["gol", "wator"]
    for p in parts:
        t0 = time.time()
        f = {"gol": make_gol, "wator": make_wator}[p]()
        print(f"wrote {f} ({f.stat().st_size} B) in {time.time() - t0:.0f} s", flush=True)
