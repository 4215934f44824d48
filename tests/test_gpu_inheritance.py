"""Inheritance and parallel_do over subtypes:
SURVEY §8(f) NEXT-3.  Expected values are closed forms of the definitions:
parallel_do<T> visits T and its subtypes, inherited fields are the leading
columns of every subtype and are addressed through any handle, objects
created during a pass are not visited -- also when they are of a subtype
whose body runs later in the same pass."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TF = [[4, 4], [4, 4, 8], [4, 4, 1], [4, 4, 8, 4]]   # Base{id, acc}; Sub1: Base+{u64}; Sub2: Base+{u8}; Sub3: Sub1+{u32}
PARENTS = [None, 0, 0, 1]
ANCESTORS = {0: {0}, 1: {0, 1}, 2: {0, 2}, 3: {0, 1, 3}}     # is_a sets


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build, dsr
    build.build()
    return dsr


def own_sum(i, T):
    v = 0
    for f in range(2, len(TF[T])):
        x = i * (f + 1)
        v += x if TF[T][f] >= 8 else x & ((1 << (8 * TF[T][f])) - 1)
    return v


def test_subtype_dispatch_and_base_field_access(D):
    n = 100003
    heap = D.Heap(TF, 1 << 26, parents=PARENTS)
    handles = torch.zeros(n, dtype=torch.int64, device="cuda")
    vals = torch.zeros(n, dtype=torch.int64, device="cuda")
    out = torch.zeros(8, dtype=torch.int64, device="cuda")
    a = D.InhArgs(handles.data_ptr(), 4, 1 << 24, out.data_ptr(), vals.data_ptr())
    heap.launch(D.K_INH_NEW, n, a)
    ids = np.arange(n)
    T = ids % 4
    assert [heap.live_count(t) for t in range(4)] == [int((T == t).sum()) for t in range(4)]
    # passes over subtrees: Sub1 (types 1, 3), Base (all), Sub3, Sub2
    acc = np.zeros(n, dtype=np.uint64)
    for root in (1, 0, 3, 2):
        heap.parallel_do(root, D.M_INH_BUMP, a)
        hit = np.array([root in ANCESTORS[t] for t in T])
        acc = np.where(hit, (3 * acc + ids.astype(np.uint64)) & 0xFFFFFFFF, acc)
    heap.launch(D.K_INH_READ, n, a)
    v = vals.cpu().numpy().view(np.uint64)
    assert np.array_equal(v & 0xFFFFFFFF, acc)                          # inherited column via any handle
    for t in range(4):
        want = sum(1 << (32 + k) for k in ANCESTORS[t])
        assert np.all((v[T == t] >> 32) << 32 == want), t               # instance-of up the parent chain
    heap.parallel_do(0, D.M_INH_SUM, a)
    o = out.cpu().numpy().view(np.uint64)
    for t in range(4):
        sel = T == t
        assert int(o[2 * t]) == int(sel.sum())
        assert int(o[2 * t + 1]) == int(acc[sel].sum()) + sum(own_sum(int(i), t) for i in ids[sel])
    assert heap.check_invariants() == 0


def test_subtree_pass_snapshot_excludes_new_objects_of_later_subtypes(D):
    """M_INH_SPAWN creates, for every visited object of type T, one object of
    type (T+1) % 4 -- whose body may run later in the same parallel_do<Base>.
    Every type's block list is built before the first body, so exactly the
    pre-pass objects are visited."""
    n = 50000
    heap = D.Heap(TF, 1 << 26, parents=PARENTS)
    handles = torch.zeros(n, dtype=torch.int64, device="cuda")
    out = torch.zeros(8, dtype=torch.int64, device="cuda")
    a = D.InhArgs(handles.data_ptr(), 4, 1 << 24, out.data_ptr(), 0)
    heap.launch(D.K_INH_NEW, n, a)
    before = [heap.live_count(t) for t in range(4)]
    heap.parallel_do(0, D.M_INH_SPAWN, a)
    assert int(out[0].item()) == n
    after = [heap.live_count(t) for t in range(4)]
    assert after == [before[t] + before[(t - 1) % 4] for t in range(4)]
    # a pass over Sub1 only spawns from types 1 and 3 (into 2 and 0)
    out.zero_()
    heap.parallel_do(1, D.M_INH_SPAWN, a)
    assert int(out[0].item()) == after[1] + after[3]
    assert heap.poll_error() == D.OK
    assert heap.check_invariants() == 0
