"""The paper's static-allocation baselines for
Game of Life and N-body (Wa-Tor's is tests/test_gpu_wator_static.py): the
same computations on plain SOA arrays, no heap.  GoL against the oracle's
textbook Life; N-body bit for bit against the heap version and at BASELINE
configs[2] against the oracle golden."""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build
    build.build()
    import paper_1810_11765_b200 as pkg
    return pkg


@pytest.mark.parametrize("W,H,p,seed,gens", [(64, 64, 0.3, 1, 100), (37, 23, 0.4, 4, 61), (3, 3, 0.5, 6, 9),
                                             (513, 385, 0.25, 7, 50), (128, 8, 0.35, 8, 30)])
def test_gol_static_equals_dense_life(P, O, W, H, p, seed, gens):
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLifeStatic
    a0 = I.gol_soup(W, H, p, seed)
    g = GameOfLifeStatic(a0)
    g.run(gens)
    assert np.array_equal(g.alive(), O.life_dense(a0, gens))


def test_gol_static_glider_and_object_version(P, O):
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLife, GameOfLifeStatic
    a0 = I.gol_pattern("glider")
    g = GameOfLifeStatic(a0)
    g.run(4 * 64)                                      # a glider crosses the 64^2 torus in 256 generations
    assert np.array_equal(g.alive(), a0)
    b0 = I.gol_soup(700, 300, 0.3, 3)
    s, o = GameOfLifeStatic(b0), GameOfLife(b0)
    for _ in range(5):
        s.run(7)
        o.run(7)
        assert np.array_equal(s.alive(), o.alive())


@pytest.mark.parametrize("n,steps,merges", [(2048, 10, True), (4096, 6, False), (1000, 10, True), (257, 5, True)])
def test_nbody_static_equals_heap_version_bit_exact(P, n, steps, merges):
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.nbody import NBody, NBodyStatic
    st = I.nbody_init(n, seed=7)
    prm = dict(G=2e-9, dt=0.5, eps=0.01, R=0.02 if merges else 1e-3)
    a = NBody(st, merges=merges, **prm)
    b = NBodyStatic(st, merges=merges, **prm)
    for _ in range(steps):
        a.run(1)
        b.run(1)
        sa, sb = a.state(), b.state()
        for k in ("alive", "x", "y", "vx", "vy", "m"):
            assert np.array_equal(sa[k], sb[k]), k
    if merges and n >= 1000:
        assert (sa["alive"] == 0).sum() > 0


def test_nbody_static_65536_ten_steps_against_golden(P):
    """BASELINE configs[2] (NBODY_PARAMS) for 10 steps: the static baseline
    meets the same oracle golden as the heap version."""
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.nbody import NBodyStatic
    g = np.load(Path(__file__).parent / "golden" / "nbody65536_10steps.npz")
    st = I.nbody_init(65536, seed=7)
    b = NBodyStatic(st, merges=True, **I.NBODY_PARAMS)
    b.run(10)
    got = b.state()
    assert np.array_equal(got["alive"], g["alive"])
    al = g["alive"] == 1
    for k in ("x", "y"):
        den = np.maximum(np.maximum(np.abs(got[k][al]), np.abs(g[k][al])), 1e-3)
        assert float(np.max(np.abs(got[k][al].astype(np.float64) - g[k][al]) / den)) <= 1e-4
