"""Full-length BASELINE runs against the oracle.

Default suite (goldens written by scripts/make_fulllength_goldens.py and
scripts/make_nbody_golden.py, which call only oracle/):

* configs[3]: Game of Life 16384^2 (p = 0.25, seed 42) for the full 1000
  generations, compared on three sampled 96 x 96 windows with the oracle's
  dense Life run on each window's 1000-generation light cone (a window of w
  cells needs the initial (w + 2 G)^2 region; errors from the region's torus
  wrap travel one cell per generation, so the inner w x w cells are exact).
* configs[1]: Wa-Tor 2048^2 for the full 500 steps: every step's event
  counters and live counts, and the final state's SHA-256, against the object
  oracle's.
* configs[2]: N-body 65,536 bodies for the full 1000 steps: the oracle state
  at step 10 (BASELINE's tolerance point), then mass conservation (<= 1e-5
  relative, BASELINE) and momentum conservation at step 1000.

The GoL run is checked for the block-list passes and for the bench's variant
(tiled prepare passes); with DSR_FULL=1 the other GoL variants (bit mirror,
all passes tiled) run the same windows, and the Wa-Tor run is also checked against the oracle recomputed live
(minutes of CPU) and against the static baseline.
"""
import hashlib
import os
from pathlib import Path

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu]
FULL = pytest.mark.skipif(os.environ.get("DSR_FULL") != "1", reason="extra full-length run: set DSR_FULL=1")
GOLDEN = Path(__file__).parent / "golden"
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build
    build.build()
    import paper_1810_11765_b200 as pkg
    return pkg


@pytest.mark.parametrize("variant", ["handles", "tiled", pytest.param("bits", marks=FULL),
                                     pytest.param("tiled_all", marks=FULL)])
def test_gol_16384_1000_generations_windows(P, variant):
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLife
    g0 = np.load(GOLDEN / "gol16384_1000gen_windows.npz")
    W, H, seed, G, w = (int(v) for v in g0["meta"])
    assert (W, H, seed, G, w) == (16384, 16384, 42, 1000, 96) and float(g0["p"][0]) == 0.25
    kw = {"handles": {}, "bits": {"bit_mirror": True}, "tiled": {"tiled": "prepare"}, "tiled_all": {"tiled": "all"}}
    g = GameOfLife(I.gol_soup(W, H, 0.25, seed), **kw[variant])
    g.run(G)
    got = g.alive()
    # window origins: numpy PCG64 seed 1 (the draws the golden script made)
    rng = np.random.default_rng(1)
    wins = [(int(rng.integers(0, H)), int(rng.integers(0, W))) for _ in range(3)]
    assert wins == [tuple(int(v) for v in r) for r in g0["windows"]]
    for (y, x), want in zip(wins, g0["alive"]):
        have = got[np.ix_(np.arange(y, y + w) % H, np.arange(x, x + w) % W)]
        assert np.array_equal(have, want), (y, x)
    assert g.heap.check_invariants() == 0


def digest(x, dtype):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.dtype(dtype).newbyteorder("<")).tobytes()).hexdigest()


def test_wator_2048_500_steps_golden(P):
    from paper_1810_11765_b200 import inputs as I, wator
    g0 = np.load(GOLDEN / "wator2048_500steps.npz")
    assert list(g0["meta"]) == [2048, 2048, 42, 500, 6, 12, 6]
    c = g0["counters"]
    WT = dict(FB=6, SB=12, SS=6, seed=42)
    kind, egg, en = I.wator_init(2048, 2048, seed=42)
    sim = wator.WaTor(kind, egg, en, **WT)
    prev = [0, 0, 0, 0]
    for s in range(500):
        sim.step()
        cur = sim.read_counters()
        assert [a - b for a, b in zip(cur, prev)] == [int(c[s, j]) for j in (2, 3, 4, 5)], f"step {s}"
        prev = cur
        if s % 50 == 49:
            assert sim.heap.live_count(0) == int(c[s, 0]) and sim.heap.live_count(1) == int(c[s, 1]), f"step {s}"
    gk, ge, gn = sim.state()
    assert [digest(gk, np.uint8), digest(ge, np.uint32), digest(gn, np.uint32)] == [str(d) for d in g0["digests"]]
    assert sim.heap.check_invariants() == 0


@FULL
def test_wator_2048_500_steps(P, O):
    from paper_1810_11765_b200 import inputs as I, wator
    WT = dict(FB=6, SB=12, SS=6, seed=42)
    kind, egg, en = I.wator_init(2048, 2048, seed=42)
    sim = wator.WaTor(kind, egg, en, **WT)
    k, e, n, c = O.wator_run(kind, egg, en, steps=500, **WT)
    prev = [0, 0, 0, 0]
    for s in range(500):
        sim.step()
        cur = sim.read_counters()
        assert [a - b for a, b in zip(cur, prev)] == [int(c[s, j]) for j in (2, 3, 4, 5)], f"step {s}"
        prev = cur
    gk, ge, gn = sim.state()
    assert np.array_equal(gk, k) and np.array_equal(ge, e) and np.array_equal(gn, n)
    assert sim.heap.live_count(0) == int(c[-1, 0]) and sim.heap.live_count(1) == int(c[-1, 1])
    assert sim.heap.check_invariants() == 0
    base = wator.WaTorStatic(kind, egg, en, **WT)
    base.run(500)
    for x, y in zip(base.state(), (k, e, n)):
        assert np.array_equal(x, y)


def test_nbody_65536_1000_steps_conservation(P):
    from paper_1810_11765_b200 import inputs as I, nbody
    g0 = np.load(GOLDEN / "nbody65536_10steps.npz")
    assert list(g0["meta"]) == [65536, 7, 10]
    st = I.nbody_init(65536, seed=7)
    prm = dict(I.NBODY_PARAMS)
    sim = nbody.NBody(st, merges=True, **prm)
    sim.run(10)
    got = sim.state()
    assert np.array_equal(got["alive"], g0["alive"])
    al = g0["alive"] == 1
    for q in ("x", "y"):
        a, b = got[q][al].astype(np.float64), g0[q][al].astype(np.float64)
        assert float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-3))) <= 1e-4
    m0 = float(np.sum(st["m"], dtype=np.float64))
    sim.run(990)
    s = sim.state()
    alive = s["alive"] == 1
    m = s["m"][alive].astype(np.float64)
    assert abs(m.sum() - m0) / m0 <= 1e-5
    # momentum starts at 0 (v = 0); pairwise forces and merges conserve it up to
    # fp32 rounding: |sum m v| stays small next to sum m |v|
    px = float(np.sum(m * s["vx"][alive])); py = float(np.sum(m * s["vy"][alive]))
    scale = float(np.sum(m * np.hypot(s["vx"][alive], s["vy"][alive])))
    print(f"N-body 1000 steps: {int(alive.sum())} bodies, mass drift {abs(m.sum() - m0) / m0:.2e}, "
          f"|P| / sum m|v| = {np.hypot(px, py) / scale:.2e}")
    assert np.hypot(px, py) <= 1e-2 * scale
    assert alive.sum() < 65536
    assert sim.heap.live_count(0) == int(alive.sum())
    assert sim.heap.check_invariants() == 0
