"""Pins of the oracle's data structures against what the paper and the
mathematics fix (no GPU).  Each test names the passage it checks."""
import random

import numpy as np
import pytest

from conftest import golden, split_fields

pytestmark = pytest.mark.filterwarnings("ignore")


# ------------------------------------------------------------------ RNG
def test_rng_splitmix64_reference_vector(O):
    g = golden("splitmix64.json")
    gamma = int(g["gamma"], 16)
    state = g["seed"]
    for want in g["outputs"]:
        assert O.sm(state) == int(want)
        state = (state + gamma) & (2**64 - 1)


def test_rng_key_composition_matches_definition(O):
    # key(seed,step,phase,idx) = sm(sm(sm(seed)^step) ^ (phase<<40 | idx)): built
    # here from the pinned sm() so a wrong composition order in or_key fails.
    for seed, step, ph, idx in [(1, 2, 3, 4), (42, 0, 0, 12345), (7, 999, 5, (1 << 40) - 1)]:
        want = O.sm(O.sm(O.sm(seed) ^ step) ^ ((ph << 40) | idx))
        assert O.key(seed, step, ph, idx) == want
    # and the input generator's numpy copy agrees with the C oracle
    from paper_1810_11765_b200 import inputs as I
    assert int(I.key(42, 3, 2, 77)) == O.key(42, 3, 2, 77)


# ------------------------------------------------------------------ layout
def test_capacity_formula_table1(O):
    g = golden("capacity.json")
    for case in g["cases"]:
        L = O.layout([split_fields(s) for s in case["sizes"]], 1 << 26)
        assert L["cap"] == case["caps"], case
    for sizes in g["too_large"]:
        with pytest.raises(ValueError):
            O.layout([split_fields(s) for s in sizes], 1 << 26)


def test_layout_worked_examples(O):
    """Hand-worked layouts (tests/golden/layout_worked.json: N_T P:308, SOA
    columns P:293, equal-size blocks P:303, per-block state P:291-293, P:464,
    P:346-352, reading R-LAYOUT) for the three BASELINE apps' type sets."""
    for c in golden("layout_worked.json")["cases"]:
        L = O.layout(c["fields"], c["heap_bytes"])
        assert L["cap"] == c["cap"], c["name"]
        assert L["col_off"] == c["col_off"], c["name"]
        assert L["block_bytes"] == c["block_bytes"], c["name"]
        assert L["M"] == c["M"], c["name"]


def test_layout_columns_are_disjoint_aligned_and_fit(O):
    rnd = random.Random(5)
    for _ in range(200):
        T = rnd.randint(1, 6)
        tf = [[rnd.choice([1, 2, 4, 8, 16]) for _ in range(rnd.randint(1, 8))] for _ in range(T)]
        sizes = [sum(f) for f in tf]
        if max(sizes) > 64 * min(sizes):
            continue
        heap = rnd.choice([1 << 20, 1 << 24, 3 << 22])
        L = O.layout(tf, heap)
        for t in range(T):
            cap = L["cap"][t]
            assert cap == 64 * min(sizes) // sizes[t]
            spans = []
            for f, s in enumerate(tf[t]):
                off = L["col_off"][t][f]
                colb = cap * s
                assert off % 16 == 0                                    # R-LAYOUT (16-B vector loads)
                if f:
                    prev_end = L["col_off"][t][f - 1] + cap * tf[t][f - 1]
                    assert prev_end <= off < prev_end + 16              # packed in declaration order
                spans.append((off, off + colb))
            assert spans[-1][1] <= L["block_bytes"]
        assert L["block_bytes"] % 128 == 0
        assert L["block_bytes"] - 128 < max(L["col_off"][t][-1] + L["cap"][t] * tf[t][-1] for t in range(T))
        # the per-block state of M blocks fits in the heap, that of M + 1 does not
        per_block_bits = 8 * (L["block_bytes"] + 21) + 1 + 2 * T
        assert L["M"] * per_block_bits <= 8 * heap < (L["M"] + 1) * per_block_bits
        # level sizes: ceil(n/64) per level until n <= 64
        n, lw = L["M"], []
        while True:
            lw.append((n + 63) // 64)
            if n <= 64:
                break
            n = (n + 63) // 64
        assert L["level_words"] == lw


# ------------------------------------------------------------------ bitmap
def test_fig7_cascade(O):
    g = golden("fig7_cascade.json")
    b = O.Bitmap(g["N"], g["W"])
    assert b.nlevels() == len(g["level_sizes"])
    for pos in g["initially_set"]:
        b.set(pos)
    assert b.consistent()
    b.trace(True)
    b.clear(g["op"][1])
    assert [list(t) for t in b.trace_get()] == g["expected_trace"]
    assert b.consistent() and b.error() == 0


@pytest.mark.parametrize("n,levels", [(1, 1), (64, 1), (65, 2), (4096, 2), (4097, 3), (262144, 3), (262145, 4)])
def test_level_count(O, n, levels):
    # nested bitmap only "if N > 64" (reading C1)
    assert O.Bitmap(n).nlevels() == levels


def _naive_consistent(b, n):
    words = [b.words(l) for l in range(b.nlevels())]
    for l in range(len(words) - 1):
        for i, w in enumerate(words[l]):
            up = (int(words[l + 1][i // 64]) >> (i % 64)) & 1
            if (int(w) != 0) != bool(up):
                return False
    return True


@pytest.mark.parametrize("n", [64, 1000, 5000, 70000])
def test_random_legal_ops_keep_consistency(O, n):
    # Appendix A: any legal multiset of set/clear keeps b^{l+1} = OR(C^l)
    rnd = random.Random(n)
    b = O.Bitmap(n)
    ref = np.zeros(n, dtype=bool)
    for _ in range(20000 if n > 1000 else 5000):
        pos = rnd.randrange(n)
        if ref[pos]:
            assert b.try_clear(pos)
            ref[pos] = False
        else:
            assert b.try_set(pos)
            ref[pos] = True
        if rnd.random() < 0.05:
            assert not (b.try_set(pos) if ref[pos] else b.try_clear(pos))   # no-op on a settled bit
    assert b.consistent() and _naive_consistent(b, n)
    assert np.array_equal(np.sort(b.indices()), np.nonzero(ref)[0].astype(np.uint64))   # Alg. 5 == naive scan
    f = b.try_find_set()
    if ref.any():
        assert f == int(np.nonzero(ref)[0][0])     # NoShift top-down ffs = lowest set bit
    else:
        assert f == -1


def test_indices_large_random(O):
    n = 1 << 21
    rng = np.random.default_rng(3)
    b = O.Bitmap(n)
    ref = np.zeros(n, dtype=bool)
    for pos in rng.choice(n, 20000, replace=False):
        b.set(int(pos))
        ref[pos] = True
    got = b.indices()
    assert len(got) == ref.sum()
    assert np.array_equal(np.sort(got), np.nonzero(ref)[0].astype(np.uint64))


def test_clear_any_drains_a_permutation(O):
    n = 3000
    b = O.Bitmap(n)
    rnd = random.Random(1)
    setb = set(rnd.sample(range(n), 700))
    for p in setb:
        b.set(p)
    got = []
    while True:
        i = b.clear_any()
        if i < 0:
            break
        got.append(i)
    assert sorted(got) == sorted(setb) and len(set(got)) == len(got)
    assert b.consistent() and b.indices().size == 0


def test_all_set_padding_and_illegal_use(O):
    b = O.Bitmap(100, all_set=True)
    assert sorted(b.indices().tolist()) == list(range(100))     # bits >= N stay 0 (C2)
    assert b.consistent()
    b.set(5)                                                      # second net set is illegal
    assert b.error() == 1


# ------------------------------------------------------------------ handles
def test_handle_listing2_masks(O):
    g = golden("listing2_masks.json")
    sm_, bm, cm = int(g["slot_mask"], 16), int(g["block_mask"], 16), int(g["cap_mask"], 16)
    rnd = random.Random(2)
    for _ in range(2000):
        t, cap, bid, slot = rnd.randint(1, 255), rnd.randint(1, 64), rnd.randrange(1 << 44), 0
        slot = rnd.randrange(cap)
        h = O.handle_encode(t, cap, bid, slot)
        assert h & sm_ == slot
        assert (h & bm) >> 6 == bid
        assert ((h & cm) >> g["cap_shift"]) + 1 == cap
        assert h >> g["type_shift"] == t
        assert O.handle_decode(h) == (t, cap, bid, slot)


# ------------------------------------------------------------------ thread assignment
def test_fig6_assignment(O):
    g = golden("fig6_assignment.json")
    for c in g["cases"]:
        nb = O.assign_num_blocks(g["r"], g["NT"], g["n"], c["tid"])
        assert nb == c["num_blocks"]
        assert [O.assign_block_pos(g["NT"], g["n"], c["tid"], k) for k in range(nb)] == c["R_positions"]
        assert O.assign_slot(g["NT"], g["n"], c["tid"], 0) == c["slot"]


def test_assignment_exact_cover(O):
    # every (block, slot) of R x [0, N_T) is assigned to exactly one (tid, k);
    # the paper's id_O = tid % N_T holds for every k iff n = 0 (mod N_T) (C9)
    rnd = random.Random(9)
    for _ in range(300):
        r, NT = rnd.randint(0, 12), rnd.randint(1, 64)
        n = rnd.choice([NT * rnd.randint(1, 6), rnd.randint(1, 300)])
        seen = {}
        for tid in range(n):
            for k in range(O.assign_num_blocks(r, NT, n, tid)):
                key = (O.assign_block_pos(NT, n, tid, k), O.assign_slot(NT, n, tid, k))
                assert key not in seen
                seen[key] = tid
                if n % NT == 0:
                    assert key[1] == tid % NT
        assert set(seen) == {(b, s) for b in range(r) for s in range(NT)}
