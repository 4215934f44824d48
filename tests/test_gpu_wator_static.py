"""GPU parity of the static-allocation Wa-Tor baseline (P:763,
dsr_wator_static_step) against the oracle, and against the object version
on the BASELINE configs[1] grid."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

WT = dict(FB=6, SB=12, SS=6, seed=42)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build
    build.build()
    import paper_1810_11765_b200 as pkg
    return pkg


@pytest.mark.parametrize("W,H,seed", [(64, 64, 5), (48, 32, 9), (203, 121, 3), (3, 3, 1)])
def test_static_every_step_bit_exact(P, O, W, H, seed):
    """Every step's state and event counters equal the oracle's (object
    oracle, the one the heap version is pinned to); odd sizes leave a ragged
    tail in the 4-cell request words."""
    from paper_1810_11765_b200 import inputs as I, wator
    kind, egg, en = I.wator_init(W, H, seed=seed)
    sim = wator.WaTorStatic(kind, egg, en, **WT)
    k, e, n = kind, egg, en
    prev = [0, 0, 0, 0]
    for s in range(60):
        k, e, n, c = O.wator_run(k, e, n, steps=1, step0=s, **WT)
        sim.run(1)
        gk, ge, gn = sim.state()
        assert np.array_equal(gk, k) and np.array_equal(ge, e) and np.array_equal(gn, n), f"step {s}"
        cur = sim.read_counters()
        assert [a - b for a, b in zip(cur, prev)] == [int(c[0, 2]), int(c[0, 3]), int(c[0, 4]), int(c[0, 5])]
        prev = cur
    # scratch arrays are left as the contract says (ready for the next call)
    assert bool((sim.target == -1).all()) and int(sim.req.sum()) == 0


def test_static_multi_step_call_equals_oracle(P, O):
    from paper_1810_11765_b200 import inputs as I, wator
    kind, egg, en = I.wator_init(160, 96, seed=21)
    sim = wator.WaTorStatic(kind, egg, en, **WT)
    sim.run(37)
    k, e, n, c = O.wator_run(kind, egg, en, steps=37, **WT)
    gk, ge, gn = sim.state()
    assert np.array_equal(gk, k) and np.array_equal(ge, e) and np.array_equal(gn, n)
    assert sim.read_counters() == [int(c[:, j].sum()) for j in (2, 3, 4, 5)]


def test_static_equals_object_version_2048(P):
    """BASELINE configs[1] grid: the baseline and the heap version agree for 100 steps."""
    from paper_1810_11765_b200 import inputs as I, wator
    kind, egg, en = I.wator_init(2048, 2048, seed=42)
    a = wator.WaTor(kind, egg, en, **WT)
    b = wator.WaTorStatic(kind, egg, en, **WT)
    for _ in range(4):
        a.run(25)
        b.run(25)
        for x, y in zip(a.state(), b.state()):
            assert np.array_equal(x, y)
    assert a.read_counters() == b.read_counters()


def test_static_rejects_bad_arguments(P):
    from paper_1810_11765_b200 import dsr
    import ctypes as C
    args = dsr.WatorStaticArgs()
    assert dsr.lib().dsr_wator_static_step(C.byref(args), 1, None) == dsr.ERR_INVALID
    assert dsr.lib().dsr_wator_static_step(None, 1, None) == dsr.ERR_INVALID
