"""Full-length BASELINE runs against the oracle (minutes each, so they run only
with DSR_FULL=1; scripts/gpu_fulllength.sh records them under profiles/):

* configs[3]: Game of Life 16384^2 (p = 0.25, seed 42) for the full 1000
  generations, compared with the oracle's dense Life on sampled windows whose
  1000-generation light cone is included (a window of w cells needs the
  initial (w + 2 G)^2 region; errors from the region's torus wrap travel one
  cell per generation, so the inner w x w cells are exact).
* configs[1]: Wa-Tor 2048^2 for the full 500 steps, every step's event
  counters and the final state against the object oracle.
* configs[2]: N-body 65,536 bodies, 1000 steps on the GPU; mass conservation
  (<= 1e-5 relative, BASELINE) and momentum conservation of the fp32 run, and
  the oracle comparison at step 10 (BASELINE's tolerance point).
"""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(os.environ.get("DSR_FULL") != "1", reason="full-length run: set DSR_FULL=1")]
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build
    build.build()
    import paper_1810_11765_b200 as pkg
    return pkg


@pytest.mark.parametrize("bit_mirror", [False, True])
def test_gol_16384_1000_generations_windows(P, O, bit_mirror):
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLife
    W = H = 16384
    G, w = 1000, 96
    a0 = I.gol_soup(W, H, 0.25, 42)
    g = GameOfLife(a0, bit_mirror=bit_mirror)
    g.run(G)
    got = g.alive()
    rng = np.random.default_rng(1)
    for _ in range(3):
        y, x = int(rng.integers(0, H)), int(rng.integers(0, W))
        ys = np.arange(y - G, y + w + G) % H
        xs = np.arange(x - G, x + w + G) % W
        region = np.ascontiguousarray(a0[np.ix_(ys, xs)])
        want = O.life_dense(region, G)[G:G + w, G:G + w]
        have = got[np.ix_(np.arange(y, y + w) % H, np.arange(x, x + w) % W)]
        assert np.array_equal(have, want), (y, x)
    assert g.heap.check_invariants() == 0


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


def test_nbody_65536_1000_steps_conservation(P, O):
    from paper_1810_11765_b200 import inputs as I, nbody
    st = I.nbody_init(65536, seed=7)
    prm = dict(I.NBODY_PARAMS)
    sim = nbody.NBody(st, merges=True, **prm)
    sim.run(10)
    got = sim.state()
    want = O.nbody_run(st, merges=True, steps=10, **prm)
    assert np.array_equal(got["alive"], want["alive"])
    al = want["alive"] == 1
    for q in ("x", "y"):
        a, b = got[q][al].astype(np.float64), want[q][al].astype(np.float64)
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
