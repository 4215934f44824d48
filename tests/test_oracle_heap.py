"""Pins of the oracle's sequential paper-heap model (Algs. 1, 2, 6-9) against
the state machine and invariants the paper fixes (no GPU)."""
import random

import numpy as np
import pytest

from conftest import split_fields

ALL = (1 << 64) - 1


def valid_mask(cap):
    return ALL if cap == 64 else (1 << cap) - 1


def check_quiescent_invariants(O, h, caps, ledger):
    """SURVEY c.7 'Allocator (concurrent)' invariants, from P:346-355, P:507,
    P:978, P:1087-1108 and Algs. 1, 2, 9."""
    M = h.M
    free = h.bitmap(0)
    assert free.consistent()
    owner = np.full(M, -1)
    fb = np.array([free.get(b) for b in range(M)])
    bm = h.alloc_bm_array()
    ty = h.type_array()
    for t, cap in enumerate(caps):
        al, ac = h.bitmap(1, t), h.bitmap(2, t)
        assert al.consistent() and ac.consistent()
        al_set = al.indices()
        ac_set = set(ac.indices().tolist())
        assert ac_set <= set(al_set.tolist())                      # active subset of allocated
        for b in al_set:
            b = int(b)
            assert owner[b] == -1 and not fb[b]                    # partition
            owner[b] = t
            assert ty[b] == t + 1                                  # type id of the block
            w = int(bm[b])
            assert (w | valid_mask(cap)) == ALL                    # padding bits set
            assert w & valid_mask(cap) != 0                        # no empty allocated block
            assert (b in ac_set) == (w != ALL)                     # active iff non-full
        live = sum(bin(int(bm[b]) & valid_mask(cap)).count("1") for b in al_set)
        assert live == h.live(t) == sum(1 for v in ledger.values() if v == t)
    for b in range(M):
        if owner[b] == -1:
            assert fb[b]                                           # free or allocated, never both/neither
            assert int(bm[b]) == ALL                               # invalidated / uninitialised
    assert h.error() == 0


def decode(O, hd):
    return O.handle_decode(hd)


def heap_of(O, tf, heap_bytes):
    """The sequential heap with as many blocks as the paper's layout bound gives heap_bytes."""
    return O.PaperHeap(tf, O.layout(tf, heap_bytes)["M"])


@pytest.mark.parametrize("sizes", [[12, 16, 24], [4, 4 * 64], [8, 16], [5, 8], [4]])
def test_random_alloc_free_sequences(O, sizes):
    tf = [split_fields(s) for s in sizes]
    L = O.layout(tf, 1 << 20)
    caps = L["cap"]
    h = heap_of(O, tf, 1 << 20)
    rnd = random.Random(sum(sizes))
    ledger = {}
    for step in range(6000):
        if ledger and (rnd.random() < 0.45 or len(ledger) > 3000):
            hd = rnd.choice(list(ledger))
            assert h.dealloc(hd) == 0
            del ledger[hd]
        else:
            t = rnd.randrange(len(sizes))
            hd = h.alloc(t)
            assert hd != 0
            assert hd not in ledger                                    # uniqueness
            ty, cap, bid, slot = decode(O, hd)
            assert ty == t + 1 and cap == caps[t] and slot < cap and bid < h.M
            ledger[hd] = t
        if step % 1000 == 999:
            check_quiescent_invariants(O, h, caps, ledger)
    for hd in list(ledger):
        h.dealloc(hd)
        del ledger[hd]
    check_quiescent_invariants(O, h, caps, ledger)
    assert h.fragmentation() == 0.0
    assert sorted(h.bitmap(0).indices().tolist()) == list(range(h.M))  # full drain


def test_dense_fill_and_state_machine(O):
    # single-threaded allocation: K <= N_T objects occupy one block; K*N_T
    # objects exactly K blocks ("allocates new objects in already
    # existing, non-full blocks")
    tf = [[4, 4, 4], [4, 4, 4, 4], [4] * 6]
    caps = [64, 48, 32]
    for t, cap in enumerate(caps):
        h = heap_of(O, tf, 1 << 20)
        hs = [h.alloc(t) for _ in range(cap)]
        bids = {decode(O, x)[2] for x in hs}
        assert len(bids) == 1
        b = bids.pop()
        assert h.alloc_bm(b) == ALL                                   # FULL
        assert h.bitmap(2, t).indices().size == 0                     # inactive when full (Alg. 1 l.12)
        assert h.bitmap(1, t).indices().tolist() == [b]
        h.dealloc(hs[0])                                              # FIRST -> active again (Alg. 2 l.5)
        assert h.bitmap(2, t).indices().tolist() == [b]
        for x in hs[1:]:
            h.dealloc(x)                                              # EMPTY -> invalidate -> free
        assert h.alloc_bm(b) == ALL
        assert h.bitmap(1, t).indices().size == 0 and h.bitmap(2, t).indices().size == 0
        assert h.bitmap(0).get(b)
        h2 = heap_of(O, tf, 1 << 20)
        K = 5
        hs = [h2.alloc(t) for _ in range(K * cap)]
        assert len({decode(O, x)[2] for x in hs}) == K


def test_capacity_one_first_and_empty_together(O):
    # N_T = 1: every free is FIRST and EMPTY at once (reading C17)
    tf = [[4], [16] * 16]          # sizes 4 and 256 -> caps 64 and 1
    h = heap_of(O, tf, 1 << 20)
    hs = [h.alloc(1) for _ in range(10)]
    assert len({decode(O, x)[2] for x in hs}) == 10
    for x in hs:
        assert h.dealloc(x) == 0
    check_quiescent_invariants(O, h, [64, 1], {})


def test_block_state_machine_exhaustive_small_caps(O):
    # For N_T <= 6: for every subset S of live slots, freeing them in a random
    # order frees the block exactly when the last one goes (EMPTY), and the
    # block is active exactly while partially full (padding generalisation C5).
    for cap_t, sizes in [(1, [4, 256]), (2, [4, 128]), (3, [4, 80]), (5, [4, 48]), (6, [4, 40])]:
        tf = [split_fields(s) for s in sizes]
        assert O.layout(tf, 1 << 20)["cap"][1] == cap_t
        rnd = random.Random(cap_t)
        for subset in range(1, 1 << cap_t):
            h = heap_of(O, tf, 1 << 20)
            hs = [h.alloc(1) for _ in range(cap_t)]
            b = decode(O, hs[0])[2]
            keep = [hs[i] for i in range(cap_t) if subset >> i & 1]
            drop = [hs[i] for i in range(cap_t) if not subset >> i & 1]
            for x in drop:
                h.dealloc(x)
            assert h.bitmap(2, 1).get(b) == (len(keep) < cap_t)
            rnd.shuffle(keep)
            for i, x in enumerate(keep):
                h.dealloc(x)
                gone = i == len(keep) - 1
                assert h.bitmap(0).get(b) == gone
                assert h.bitmap(1, 1).get(b) == (not gone)
                assert h.bitmap(2, 1).get(b) == (not gone)


def test_oom_returns_null_and_linux_scalability_utilisation(O):
    # heap sized for exactly K 64-byte objects; DynaSOAr reaches
    # 96.9% utilisation.  Sequential placement must reach >= 95%.
    K = 1 << 16
    heap = K * 64
    tf = [[4] * 16]
    h = heap_of(O, tf, heap)
    n = 0
    while h.alloc(0) != 0:
        n += 1
    assert n / K >= 0.95
    assert h.alloc(0) == 0                     # still OOM (reading C14: null, not a spin)
    assert n == h.M * 64


def test_fragmentation_formula(O):
    # F = sum (N - used) / sum N over allocated blocks
    tf = [[4, 4, 4], [4, 4, 4, 4]]                 # caps 64, 48
    h = heap_of(O, tf, 1 << 20)
    a = [h.alloc(0) for _ in range(64)]
    b = [h.alloc(1) for _ in range(10)]
    assert abs(h.fragmentation() - (0 + 38) / (64 + 48)) < 1e-12
    for x in a[:32]:
        h.dealloc(x)
    assert abs(h.fragmentation() - (32 + 38) / (64 + 48)) < 1e-12
    for x in a[32:] + b:
        h.dealloc(x)
    assert h.fragmentation() == 0.0


# ------------------------------------------------------------------ scripted interleavings
# The branches of Algs. 1, 2 and 9 that only a concurrent execution reaches,
# pinned by running "another thread's" operations at the linearisation point
# where the paper says they can interleave.  The expected states are derived
# by hand from the algorithms' text, step by step, in each test's docstring.

def test_type_change_rollback_alg1_l14(O):
    """P:369 / Alg. 1 l.9-14: a thread found block b0 (type A) in
    active[A]; before its reservation, the block's last object is freed (b0 is
    invalidated and freed, Alg. 2) and another thread re-initialises b0 as
    type B (slow path: free.clear() returns the lowest free block, b0) and
    takes slot 0.  The first thread's reservation then succeeds on slot 1 of
    a type-B block, reads t = B != A and rolls back (deallocate of slot 1:
    REGULAR, b0 keeps B's object), retries, finds active[A] empty and
    initialises the next free block b1 for A."""
    tf = [[4], [4, 4]]                 # caps 64 (A) and 32 (B)
    h = O.PaperHeap(tf, 4)
    x = h.alloc(0)
    assert decode(O, x) == (1, 64, 0, 0)
    seen = {}

    def other_thread(bid):
        seen["bid"] = bid
        assert h.dealloc(x) == 0                       # b0 empties: invalidate, free.set(b0)
        seen["y"] = h.alloc(1)                         # b0 re-initialised as type B
    h.on(O.HOOK_FOUND, other_thread)
    z = h.alloc(0)
    assert seen["bid"] == 0
    assert decode(O, seen["y"]) == (2, 32, 0, 0)       # B's object in b0 slot 0
    assert decode(O, z) == (1, 64, 1, 0)               # A's object in the fresh block b1
    assert h.counters()["rollbacks"] == 1
    assert h.type(0) == 2 and h.type(1) == 1
    assert h.alloc_bm(0) == ((ALL << 32) & ALL) | 1    # B: padding bits 32..63 + slot 0 (slot 1 rolled back)
    assert h.alloc_bm(1) == 1
    assert h.bitmap(2, 0).indices().tolist() == [1] and h.bitmap(2, 1).indices().tolist() == [0]
    assert h.bitmap(1, 0).indices().tolist() == [1] and h.bitmap(1, 1).indices().tolist() == [0]
    assert sorted(h.bitmap(0).indices().tolist()) == [2, 3]
    check_quiescent_invariants(O, h, [64, 32], {seen["y"]: 1, z: 0})


def test_invalidation_fails_and_rolls_back_alg9(O):
    """Alg. 2 l.6-7 + Alg. 9 l.8-13: a thread frees the last
    object of b0 (EMPTY); before it invalidates, another thread reserves slot 0
    of b0 (still active).  The invalidation's atomicOr returns before = slot 0
    != 0: it fails, the rollback atomicAnd(before) restores exactly slot 0;
    before_rollback = ~0 (nobody freed in between), so no deferred
    deactivation, and (before_rollback & before) != 0, so no retry.  b0 stays
    allocated and active with one object."""
    tf = [[4]]
    h = O.PaperHeap(tf, 2)
    x1, x2 = h.alloc(0), h.alloc(0)
    assert h.dealloc(x1) == 0
    seen = {}
    h.on(O.HOOK_EMPTIED, lambda bid: seen.setdefault("z", h.alloc(0)))
    assert h.dealloc(x2) == 0
    assert decode(O, seen["z"]) == (1, 64, 0, 0)
    c = h.counters()
    assert c["invalidate_fail"] == 1 and c["invalidate_retry"] == 0 and c["deferred_deactivation"] == 0
    assert h.alloc_bm(0) == 1
    assert h.bitmap(2, 0).indices().tolist() == [0] and h.bitmap(1, 0).indices().tolist() == [0]
    assert h.bitmap(0).indices().tolist() == [1]
    check_quiescent_invariants(O, h, [64], {seen["z"]: 0})


def test_invalidation_rollback_deferred_deactivation_and_retry(O):
    """The paper's "Details" of Alg. 9: as above, but inside the
    invalidation window (after the atomicOr, before the rollback) the other
    thread frees its object again.  Its atomicAnd sees an all-ones bitmap:
    FIRST, so it calls active.set(b0) -- which spins, the bit still being set
    ("this set(bid) operation will spin until we deactivate the block").  The
    rollback returns before_rollback = ~1 != ~0: the deferred active.clear
    (l.10) runs, the spinning set completes; (before_rollback & before) = 0:
    empty again, so the invalidation is retried (l.12), now succeeds, and
    Alg. 2 l.8-11 frees b0.  Nothing is left allocated; the spinning op did
    not deadlock."""
    tf = [[4]]
    h = O.PaperHeap(tf, 2)
    x1, x2 = h.alloc(0), h.alloc(0)
    h.dealloc(x1)
    seen = {}

    def reserve_in_window(bid):
        seen["z"] = h.alloc(0)

    def free_in_invalidation_window(bid):
        assert bid == 0
        assert h.dealloc(seen["z"]) == 0

    h.on(O.HOOK_EMPTIED, reserve_in_window)
    h.on(O.HOOK_INVALIDATED, free_in_invalidation_window)
    assert h.dealloc(x2) == 0
    c = h.counters()
    assert c == {"rollbacks": 0, "invalidate_fail": 1, "invalidate_retry": 1, "deferred_deactivation": 1}
    assert h.alloc_bm(0) == ALL                           # invalidated = free
    assert h.bitmap(2, 0).indices().size == 0 and h.bitmap(1, 0).indices().size == 0
    assert sorted(h.bitmap(0).indices().tolist()) == [0, 1]
    check_quiescent_invariants(O, h, [64], {})


def test_spinning_set_is_the_papers_deadlock(O):
    """a second net set of a bit is illegal and spins forever; in the
    sequential model it stays pending and is reported until a clear of the
    same bit releases it (then the bitmap is consistent again)."""
    b = O.Bitmap(200)
    b.set(70)
    b.set(70)
    assert b.error() == 1
    b.clear(70)                                          # releases the waiting set
    assert b.error() == 0 and b.get(70) and b.consistent()
