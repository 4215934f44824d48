"""Pins of the oracle's SMMO workloads (no GPU): closed forms, textbook
patterns, brute force on tiny inputs, conservation laws."""
import numpy as np
import pytest

from paper_1810_11765_b200 import inputs as I


# ------------------------------------------------------------------ microbench
def mb_closed_form(seed, n1, n2):
    """Expected per-type (count, sum, xor) after phases 2 and 5 computed by a
    direct loop over t through key() with no heap (SURVEY c.7 'Microbench')."""
    nf = [3, 4, 6]

    def fields(t0, n):
        t = np.arange(t0, t0 + n, dtype=np.uint64)
        q = (t & np.uint64(3)).astype(np.int64)
        ty = np.where(q < 2, 0, np.where(q == 2, 1, 2))
        out = []
        for T in range(3):
            tt = t[ty == T]
            f = np.stack([(I.key(seed, 0, I.PH_MB_FIELD, tt * np.uint64(16) + np.uint64(k))
                           & np.uint64(0xFFFFFFFF)) for k in range(nf[T])], axis=1)
            out.append(f)
        return out

    def red(fs):
        res = []
        for f in fs:
            s = int(f.astype(np.uint64).sum(dtype=np.uint64)) if f.size else 0
            x = int(np.bitwise_xor.reduce(f.reshape(-1))) if f.size else 0
            res.append((len(f), s % (1 << 64), x))
        return res

    f1 = fields(0, n1)
    ph2 = red(f1)
    surv = [f[(f[:, 0] & np.uint64(1)) == 0] for f in f1]         # phase 3 deletes odd field0
    f4 = fields(n1, n2)
    ph5 = red([np.concatenate([a, b]) for a, b in zip(surv, f4)])
    return ph2, ph5


@pytest.mark.parametrize("n1,n2", [(1000, 500), (4096, 2048), (1 << 16, 1 << 15)])
def test_microbench_closed_form(O, n1, n2):
    out, live = O.microbench(1, n1, n2)
    ph2, ph5 = mb_closed_form(1, n1, n2)
    assert [tuple(int(v) for v in out[0, t]) for t in range(3)] == ph2
    assert [tuple(int(v) for v in out[1, t]) for t in range(3)] == ph5
    assert live[5].tolist() == [0, 0, 0]
    assert live[0].sum() == n1 and live[0][0] == (n1 + 3) // 4 + (n1 + 2) // 4


def test_microbench_permutation_invariant(O):
    a, la = O.microbench(3, 5000, 3000, order_seed=0)
    b, lb = O.microbench(3, 5000, 3000, order_seed=12345)
    assert np.array_equal(a, b) and np.array_equal(la, lb)


# ------------------------------------------------------------------ Game of Life
def test_gol_blinker_period_two(O):
    a0 = I.gol_pattern("blinker")
    a1, _ = O.gol_run(a0, 1)
    a2, _ = O.gol_run(a0, 2)
    assert not np.array_equal(a0, a1) and np.array_equal(a0, a2)
    assert a1.sum() == 3 and a1[9:12, 11].sum() == 3                  # vertical phase


@pytest.mark.parametrize("name", ["block", "beehive"])
def test_gol_still_lifes(O, name):
    a0 = I.gol_pattern(name)
    a, _ = O.gol_run(a0, 7)
    assert np.array_equal(a, a0)


def test_gol_glider_translates(O):
    a0 = I.gol_pattern("glider")
    for k in range(1, 6):
        a, _ = O.gol_run(a0, 4 * k)
        assert np.array_equal(a, np.roll(np.roll(a0, k, axis=0), k, axis=1))   # (+1,+1) per 4 gens
    a, _ = O.gol_run(a0, 4 * 64)
    assert np.array_equal(a, a0)                                                 # wraps the 64x64 torus


@pytest.mark.parametrize("W,H,p,seed", [(64, 64, 0.3, 1), (64, 64, 0.3, 2), (64, 64, 0.3, 3),
                                        (37, 23, 0.4, 4), (8, 8, 0.5, 5), (3, 3, 0.5, 6)])
def test_gol_equals_dense_life(O, W, H, p, seed):
    a0 = I.gol_soup(W, H, p, seed)
    for gens in (1, 7, 100):
        a, _ = O.gol_run(a0, gens)
        assert np.array_equal(a, O.life_dense(a0, gens)), gens


def test_gol_candidate_invariant_and_permutation(O):
    a0 = I.gol_soup(48, 40, 0.3, 11)
    _, recs = O.gol_run(a0, 30, dump=True)
    _, recs2 = O.gol_run(a0, 30, order_seed=99, dump=True)
    for g in range(30):
        assert np.array_equal(recs[g], recs2[g])                    # order-independent
        alive = np.zeros(48 * 40, bool)
        cand = np.zeros(48 * 40, bool)
        r = recs[g]
        alive[r[r[:, 1] == 1, 0]] = True
        cand[r[r[:, 1] == 2, 0]] = True
        A = alive.reshape(40, 48)
        k = sum(np.roll(np.roll(A, dy, 0), dx, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
                if dy or dx).reshape(-1)
        # every dead cell with >= 1 alive neighbour holds a Candidate
        assert np.all(cand[(~alive) & (k > 0)])
        assert not np.any(cand & alive)


# ------------------------------------------------------------------ Wa-Tor
P = dict(FB=6, SB=12, SS=6, seed=42)


def test_wator_object_equals_dense_and_ledger(O):
    kind, egg, en = I.wator_init(64, 64, seed=5)
    k1, e1, n1, c1 = O.wator_run(kind, egg, en, steps=120, **P)
    k2, e2, n2, c2 = O.wator_run(kind, egg, en, steps=120, dense=True, **P)
    assert np.array_equal(k1, k2) and np.array_equal(e1, e2) and np.array_equal(n1, n2)
    assert np.array_equal(c1, c2)
    fish, sharks = int((kind == 1).sum()), int((kind == 2).sum())
    for s in range(120):
        f, sh, bf, bs, eat, starv = (int(v) for v in c1[s])
        assert f == fish + bf - eat and sh == sharks + bs - starv      # population ledger
        fish, sharks = f, sh
    assert c1[:, 2].sum() > 0 and c1[:, 4].sum() > 0 and c1[:, 5].sum() > 0


def test_wator_permutation_invariant(O):
    kind, egg, en = I.wator_init(48, 32, seed=9)
    a = O.wator_run(kind, egg, en, steps=40, **P)
    b = O.wator_run(kind, egg, en, steps=40, order_seed=777, **P)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_wator_sharks_only_starve_on_schedule(O):
    # sharks only, egg = 0, SS < SB: no shark ever eats or breeds, so the
    # population is constant for SS - 1 steps and 0 after step SS (closed form)
    H, W = 32, 32
    kind = np.zeros((H, W), np.uint8)
    kind[::3, ::3] = 2
    n0 = int(kind.sum() // 2)
    egg = np.zeros((H, W), np.uint32)
    en = np.where(kind == 2, 6, 0).astype(np.uint32)
    _, _, _, c = O.wator_run(kind, egg, en, FB=6, SB=12, SS=6, seed=1, steps=8)
    assert c[:5, 1].tolist() == [n0] * 5
    assert c[5:, 1].tolist() == [0, 0, 0]
    assert c[:, 3].sum() == 0 and c[5, 5] == n0


def test_wator_empty_is_static_and_fish_only_conserve(O):
    z = np.zeros((16, 16), np.uint8)
    k, e, n, c = O.wator_run(z, z.astype(np.uint32), z.astype(np.uint32), steps=5, **P)
    assert k.sum() == 0 and c.sum() == 0
    # fish only: nobody is eaten, population only grows by births
    kind = np.zeros((16, 16), np.uint8)
    kind[::4, ::4] = 1
    egg = np.zeros((16, 16), np.uint32)
    k, e, n, c = O.wator_run(kind, egg, egg.copy(), steps=20, **P)
    assert c[:, 4].sum() == 0 and c[-1, 0] == 16 + c[:, 2].sum()


# ------------------------------------------------------------------ N-body
def two_body(d=0.01, m1=1.0, m2=1.0):
    return {"x": np.array([-d, d], np.float32), "y": np.zeros(2, np.float32),
            "vx": np.zeros(2, np.float32), "vy": np.zeros(2, np.float32),
            "m": np.array([m1, m2], np.float32), "alive": np.ones(2, np.uint8)}


def test_nbody_two_equal_bodies_mirror(O):
    s = O.nbody_run(two_body(), G=1e-6, dt=0.5, eps=1e-4, R=1e-5, merges=False, steps=20)
    assert s["x"][0] == -s["x"][1] and s["vx"][0] == -s["vx"][1]
    assert s["x"][0] > -0.01 and s["x"][1] < 0.01                        # attraction


def test_nbody_two_body_force_closed_form(O):
    # one step from rest: f = G m1 m2 d / (d^2 + eps^2)^{3/2}, v = f/m dt, x += v dt
    d, G, dt, eps = 0.02, 1e-6, 0.5, 1e-3
    s = O.nbody_run(two_body(d / 2), G=G, dt=dt, eps=eps, R=1e-9, merges=False, steps=1)
    f = G * d / (d * d + eps * eps) ** 1.5
    assert abs(float(s["vx"][0]) - f * dt) <= 1e-6 * f * dt
    assert abs(float(s["x"][0]) - (-d / 2 + f * dt * dt)) <= 1e-7


def test_nbody_momentum_conserved_without_merges(O):
    st = I.nbody_init(512, seed=3)
    st["vx"] = (np.random.default_rng(1).standard_normal(512) * 1e-4).astype(np.float32)
    s = O.nbody_run(st, G=1e-6, dt=0.5, eps=1e-3, R=1e-3, merges=False, steps=10)
    p0 = float((st["m"].astype(np.float64) * st["vx"]).sum())
    p1 = float((s["m"].astype(np.float64) * s["vx"]).sum())
    scale = float((st["m"].astype(np.float64) * np.abs(st["vx"])).sum())
    assert abs(p1 - p0) <= 1e-5 * scale


def test_nbody_G0_static_and_merge_set_from_geometry(O):
    st = I.nbody_init(2000, seed=4)
    R = 0.02
    s = O.nbody_run(st, G=0.0, dt=0.5, eps=1e-3, R=R, merges=True, steps=1)
    x, y, m = st["x"].astype(np.float64), st["y"].astype(np.float64), st["m"]
    n = len(x)
    # brute force: target = nearest heavier (m, id)-larger body within R
    tgt = np.full(n, -1)
    for i in range(n):
        d2 = (x - x[i]) ** 2 + (y - y[i]) ** 2
        heav = (m > m[i]) | ((m == m[i]) & (np.arange(n) > i))
        ok = heav & (d2 < R * R)
        ok[i] = False
        if ok.any():
            c = np.nonzero(ok)[0]
            tgt[i] = c[np.lexsort((c, d2[c]))[0]]
    inc = np.full(n, -1)
    for i in range(n):
        if tgt[i] >= 0 and (inc[tgt[i]] < 0 or i < inc[tgt[i]]):
            inc[tgt[i]] = i
    absorbed = {int(inc[j]) for j in range(n) if inc[j] >= 0 and tgt[j] < 0}
    assert {int(i) for i in np.nonzero(s["alive"] == 0)[0]} == absorbed
    assert len(absorbed) > 0
    # mass conserved exactly up to fp32 adds, and untouched bodies did not move
    assert abs(float(s["m"][s["alive"] == 1].astype(np.float64).sum()) - float(m.astype(np.float64).sum())) \
        <= 1e-5 * float(m.sum())
    untouched = [i for i in range(n) if i not in absorbed and inc[i] < 0 or tgt[i] >= 0 and i not in absorbed]
    for i in untouched[:200]:
        if inc[i] < 0:
            assert s["x"][i] == st["x"][i] and s["y"][i] == st["y"][i]


def test_nbody_single_merge_conserves(O):
    st = two_body(d=0.001, m1=1.0, m2=3.0)
    st["vx"] = np.array([0.5, -0.25], np.float32)
    s = O.nbody_run(st, G=0.0, dt=0.0, eps=1e-3, R=0.01, merges=True, steps=1)
    assert s["alive"].tolist() == [0, 1]
    assert s["m"][1] == np.float32(4.0)
    assert abs(float(s["vx"][1]) - (1.0 * 0.5 + 3.0 * -0.25) / 4.0) < 1e-7     # momentum
    assert abs(float(s["x"][1]) - (1.0 * -0.001 + 3.0 * 0.001) / 4.0) < 1e-9    # centre of mass
