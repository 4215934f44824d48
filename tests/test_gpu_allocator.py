"""GPU parity tests of the allocator through the C ABI (libdsr.so):
single-thread replay against the oracle's sequential paper-heap model,
concurrent torture with the quiescent invariant audit, the microbenchmark
against the oracle and its closed form, Linux Scalability utilisation."""
import ctypes as C
import random

import numpy as np
import pytest

from conftest import split_fields

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build, dsr
    build.build()
    return dsr


def words_of(oracle_bitmap, nlevels):
    return [oracle_bitmap.words(l) for l in range(nlevels)]


def compare_state(D, heap, oh, ntypes):
    M = heap.M
    assert oh.M == M
    assert np.array_equal(heap.copy_state(0), oh.alloc_bm_array())
    assert np.array_equal(heap.copy_state(1), oh.type_array())
    nl = heap.layout["nlevels"]
    for got, want in zip(heap.copy_state(2), words_of(oh.bitmap(0), nl)):
        assert np.array_equal(got, want)
    for t in range(ntypes):
        for what, which in ((3, 1), (4, 2)):
            for got, want in zip(heap.copy_state(what, t), words_of(oh.bitmap(which, t), nl)):
                assert np.array_equal(got, want), (what, t)


def replay_ops(rnd, ntypes, n, free_p=0.45):
    ops, live = [], []
    for i in range(n):
        if live and rnd.random() < free_p:
            j = live.pop(rnd.randrange(len(live)))
            ops.append((1, j))
        else:
            ops.append((0, rnd.randrange(ntypes)))
            live.append(i)
    return ops


@pytest.mark.parametrize("sizes,heap_bytes,M", [([12, 16, 24], 1 << 20, 700), ([4, 256], 1 << 20, 1037),
                                                ([5, 8], 3 << 18, 333), ([8, 8, 40, 100], 1 << 21, 3005),
                                                ([12, 16, 24], 1 << 20, 64), ([4, 8], 1 << 20, 65),
                                                ([4, 256], 1 << 20, 40)])
def test_single_thread_replay_matches_oracle(D, O, sizes, heap_bytes, M):
    """grid = 1x1, rotation and coalescing off: the CUDA allocator must produce
    the oracle's words, type ids and handles exactly (Algs. 1-9).  Both heaps
    get the same block count M ("determined at compile time"), chosen
    here (ragged, one-level and two-level bitmaps); small M also drives the
    replay into OOM (null handles) and block re-typing."""
    tf = [split_fields(s) for s in sizes]
    rnd = random.Random(sum(sizes))
    heap = D.Heap(tf, heap_bytes, flags=D.F_NO_ROTATE | D.F_NO_COALESCE | D.F_NO_HINT, max_blocks=M)
    assert heap.M == M
    oh = O.PaperHeap(tf, M)
    ops = replay_ops(rnd, len(tf), 3000)
    want = []
    for op, arg in ops:
        if op == 0:
            want.append(oh.alloc(arg))
        else:
            if want[arg]:                                       # destroy(null) is a no-op (OOM earlier)
                assert oh.dealloc(want[arg]) == 0
            want.append(0)
    flat = np.array(ops, dtype=np.uint32).reshape(-1)
    d_ops = torch.from_numpy(flat.astype(np.int32)).cuda()
    d_h = torch.zeros(len(ops), dtype=torch.int64, device="cuda")
    heap.launch(D.K_REPLAY, 1, D.ReplayArgs(d_ops.data_ptr(), len(ops), d_h.data_ptr()))
    torch.cuda.synchronize()
    got = d_h.cpu().numpy().view(np.uint64)
    assert np.array_equal(got, np.array(want, dtype=np.uint64))
    compare_state(D, heap, oh, len(tf))
    assert heap.check_invariants() == 0
    assert heap.poll_error() == (D.ERR_OOM if 0 in [w for (op, _), w in zip(ops, want) if op == 0] else D.OK)


def test_fresh_heap_state_and_invariants(D, O):
    tf = [[4, 4, 4], [4, 4, 4, 4], [4] * 6]
    heap = D.Heap(tf, 1 << 26, max_blocks=50_000)
    oh = O.PaperHeap(tf, 50_000)
    compare_state(D, heap, oh, 3)
    assert heap.check_invariants() == 0
    assert [heap.live_count(t) for t in range(3)] == [0, 0, 0]
    assert heap.fragmentation()[0] == 0.0


@pytest.mark.parametrize("flags", [0, 1, 2, 3, 16])
def test_torture_concurrent_new_destroy(D, flags):
    """Many warps call new/destroy from divergent lanes; afterwards: no canary
    damage, every quiescent invariant holds, the live set equals the ledger."""
    tf = [[4, 4, 4], [4, 4, 4, 4], [4] * 6, [4] * 16, [4, 4]]   # caps 42, 32, 21, 8, 64
    # NoShift makes every leader hit the same blocks; with failed reservations
    # counting as failed lookups (R-RETRY) it initialises many more blocks
    heap = D.Heap(tf, (1 << 27) if not flags & D.F_NO_ROTATE else (1 << 30), flags=flags | D.F_STATS)
    nthreads = 1 << 17
    ledger = torch.zeros(nthreads * 8, dtype=torch.int64, device="cuda")
    errors = torch.zeros(1, dtype=torch.int64, device="cuda")
    heap.launch(D.K_TORTURE, nthreads, D.TortureArgs(12345 + flags, 40, 1, ledger.data_ptr(), errors.data_ptr()))
    torch.cuda.synchronize()
    assert int(errors.item()) == 0
    assert heap.poll_error() == D.OK
    assert heap.check_invariants() == 0
    led = ledger.cpu().numpy().view(np.uint64)
    led = np.sort(led[led != 0])
    assert len(np.unique(led)) == len(led)                     # uniqueness
    # collect every live object through parallel_do
    got = []
    for t in range(len(tf)):
        out = torch.zeros(len(led) + 1, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        heap.parallel_do(t, D.M_COLLECT, D.CollectArgs(out.data_ptr(), cnt.data_ptr()))
        torch.cuda.synchronize()
        k = int(cnt.item())
        got.append(out[:k].cpu().numpy().view(np.uint64))
        assert heap.live_count(t) == k
    got = np.sort(np.concatenate(got))
    assert np.array_equal(got, led)
    st = heap.stats()
    assert st["allocs"] - st["frees"] == len(led)
    # drain: free everything, heap returns to all-free
    for t in range(len(tf)):
        heap.parallel_do(t, D.M_MB_FREE_ALL)
    torch.cuda.synchronize()
    assert heap.check_invariants() == 0
    assert [heap.live_count(t) for t in range(len(tf))] == [0] * len(tf)
    free_words = heap.copy_state(2)[0]
    M = heap.M
    assert int(sum(bin(int(w)).count("1") for w in free_words)) == M


def mb_expected(O, seed, n1, n2):
    out, live = O.microbench(seed, n1, n2)
    return out


@pytest.mark.parametrize("bulk", [True, False])
@pytest.mark.parametrize("n1,n2", [(1000, 500), (1 << 16, 1 << 15), (3 * 65536 + 77, 40001)])
def test_microbench_matches_oracle(D, O, n1, n2, bulk):
    from paper_1810_11765_b200.microbench import Microbench
    mb = Microbench(n1=n1, n2=n2, seed=1, bulk=bulk)
    mb.step()
    torch.cuda.synchronize()
    assert np.array_equal(mb.results(), mb_expected(O, 1, n1, n2))
    assert mb.heap.poll_error() == D.OK
    assert [mb.heap.live_count(t) for t in range(3)] == [0, 0, 0]
    assert mb.heap.check_invariants() == 0
    # a second step on the same heap (reset inside) gives the same result
    mb.step()
    assert np.array_equal(mb.results(), mb_expected(O, 1, n1, n2))


@pytest.mark.parametrize("bulk", [True, False])
def test_microbench_full_size_closed_form(D, bulk):
    """BASELINE configs[4] at full size (2^26 + 2^25 objects) in the bench's
    launch configuration, against the closed form (direct loop over t)."""
    from paper_1810_11765_b200.microbench import Microbench
    from test_oracle_apps import mb_closed_form
    n1, n2 = 1 << 26, 1 << 25
    mb = Microbench(n1=n1, n2=n2, seed=1, bulk=bulk)
    mb.step()
    torch.cuda.synchronize()
    r = mb.results()
    ph2, ph5 = mb_closed_form(1, n1, n2)
    assert [tuple(int(v) for v in r[0, t]) for t in range(3)] == ph2
    assert [tuple(int(v) for v in r[1, t]) for t in range(3)] == ph5
    assert mb.heap.poll_error() == D.OK
    assert mb.heap.check_invariants() == 0


def test_linux_scalability_utilisation(D):
    """heap sized for exactly 16384 x n 64-byte objects; DynaSOAr
    reached 96.9% utilisation.  We require >= 95% before OOM."""
    n = 64
    threads = 16384
    heap_bytes = threads * n * 64
    heap = D.Heap([[4] * 16], heap_bytes)
    handles = torch.zeros(threads * n, dtype=torch.int64, device="cuda")
    heap.launch(D.K_LS_ALLOC, threads, D.LsArgs(handles.data_ptr(), n, 0))
    torch.cuda.synchronize()
    h = handles.cpu().numpy().view(np.uint64)
    ok = int((h != 0).sum())
    assert heap.poll_error() == D.ERR_OOM                      # the heap cannot hold all of them
    assert ok / (threads * n) >= 0.95
    assert ok == heap.live_count(0)
    assert len(np.unique(h[h != 0])) == ok
    heap.launch(D.K_LS_FREE, threads, D.LsArgs(handles.data_ptr(), n, 0))
    torch.cuda.synchronize()
    assert heap.live_count(0) == 0
    assert heap.check_invariants() == 0


def test_reserve_blocks_and_trim(D):
    """dsr_reserve_blocks runs the slow path ahead of time (empty active
    blocks); a following burst of new fills them; dsr_trim returns the blocks
    that stayed empty, leaving every quiescent invariant intact."""
    tf = [[4, 4, 4], [4, 4, 4, 4]]
    heap = D.Heap(tf, 1 << 26)
    heap.reserve_blocks(0, 1000)
    heap.reserve_blocks(1, 10)
    torch.cuda.synchronize()
    _, blocks = heap.fragmentation()
    assert blocks == [1000, 10]
    assert heap.check_invariants() > 0            # empty allocated blocks exist until the trim
    n = 40000
    handles = torch.zeros(n, dtype=torch.int64, device="cuda")
    heap.launch(D.K_LS_ALLOC, n, D.LsArgs(handles.data_ptr(), 1, 0))
    heap.trim(0)
    heap.trim(1)
    torch.cuda.synchronize()
    assert heap.live_count(0) == n and heap.live_count(1) == 0
    f, blocks = heap.fragmentation()
    assert blocks[1] == 0 and blocks[0] >= -(-n // heap.cap[0])
    assert heap.check_invariants() == 0
    assert heap.poll_error() == D.OK


@pytest.mark.parametrize("reserve,flags,bulk", [(False, 0, False), (True, 0, False), (True, 32, False),
                                                (True, 0, True), (False, 1, True), (False, 2, True)])
def test_microbench_variants_match_oracle(D, O, reserve, flags, bulk):
    from paper_1810_11765_b200.microbench import Microbench
    mb = Microbench(n1=200_000, n2=100_000, seed=5, reserve=reserve, flags=flags, bulk=bulk)
    mb.step()
    assert np.array_equal(mb.results(), O.microbench(5, 200_000, 100_000)[0])
    assert mb.heap.check_invariants() == 0


@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("n1,n2", [(1 << 16, 1 << 15), (400_000, 123_458)])
def test_microbench_host_inputs_match_oracle(D, O, n1, n2, host):
    """The end-to-end form of the step (bench.py e2e): field values from
    caller arrays (inputs.mb_fields) instead of device-computed keys -- device
    arrays, or HOST arrays that dsr_launch stages through its copy stream and
    two alternating device buffers (three steps reuse them); same results as
    the oracle.  n2 not a multiple of 4: the caller passes ceil(n/4) groups."""
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.microbench import Microbench
    f1 = torch.from_numpy(I.mb_fields(1, 0, n1).view(np.int32))
    f2 = torch.from_numpy(I.mb_fields(1, n1, -(-n2 // 4) * 4).view(np.int32))
    f1, f2 = (f1.pin_memory(), f2.pin_memory()) if host else (f1.cuda(), f2.cuda())
    mb = Microbench(n1=n1, n2=n2, seed=1)
    want = O.microbench(1, n1, n2)[0]
    for _ in range(3 if host else 1):
        mb.step(inputs=(f1.data_ptr(), f2.data_ptr()), host_inputs=host)
        torch.cuda.synchronize()
        assert np.array_equal(mb.results(), want)
    assert mb.heap.check_invariants() == 0


def test_microbench_host_inputs_reject_unaligned_t0(D):
    from paper_1810_11765_b200.microbench import Microbench
    mb = Microbench(n1=4096, n2=4096, seed=1)
    buf = torch.zeros(4 * 4096, dtype=torch.int32, device="cuda")
    with pytest.raises(D.DsrError):
        mb.heap.launch(D.K_MB_NEW, 1024, D.MbNewArgs(1, 2, buf.data_ptr()))


def test_atomic_probe(D):
    """dsr_probe_atomics: both modes run and report the atomics issued; the
    same-address mode is far slower than hashed addresses (serialisation)."""
    buf = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
    rates = []
    for mode in (0, 1):
        D.probe_atomics(buf, mode, 4)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = D.probe_atomics(buf, mode, 8)
        e1.record()
        torch.cuda.synchronize()
        assert n > 0 and n % 256 == 0
        rates.append(n / e0.elapsed_time(e1))
    assert rates[0] > 10 * rates[1]
    with pytest.raises(D.DsrError):
        D.probe_atomics(buf[:1], 0, 4)


@pytest.mark.parametrize("bulk", [True, False])
@pytest.mark.parametrize("n1,n2", [(0, 0), (1, 0), (3, 1), (5, 7), (33, 31), (767, 769), (1536, 1)])
def test_microbench_degenerate_sizes(D, O, n1, n2, bulk):
    """Empty and tiny workloads (no object, one object, partial warps and
    partial type groups, ragged bulk units) give the oracle's results and
    leave the heap empty."""
    from paper_1810_11765_b200.microbench import Microbench
    mb = Microbench(n1=n1, n2=n2, seed=9, bulk=bulk)
    mb.step()
    torch.cuda.synchronize()
    assert np.array_equal(mb.results(), O.microbench(9, n1, n2)[0])
    assert mb.heap.poll_error() == D.OK
    assert [mb.heap.live_count(t) for t in range(3)] == [0, 0, 0]
    assert mb.heap.check_invariants() == 0


@pytest.mark.parametrize("bulk", [True, False])
def test_microbench_live_set_elementwise(D, O, bulk):
    """Element-wise parity of the microbench (SURVEY c.8): after phases 1, 3
    and 4 the canonical dump of every type (each live object's packed fields,
    sorted by bytes) equals the oracle object store's live set, at n1 = 2^20
    (ragged n2), with the bench's kernels."""
    from paper_1810_11765_b200.microbench import Microbench
    n1, n2 = 1 << 20, (1 << 19) + 13
    mb = Microbench(n1=n1, n2=n2, seed=1, bulk=bulk)
    for stop in (1, 3, 4):
        mb.step(stop=stop)
        torch.cuda.synchronize()
        for t in range(3):
            got = mb.heap.canonical_dump(t)
            want = O.microbench_live(1, n1, n2, stop, t)
            assert got.shape[0] == want.shape[0], (stop, t)
            assert np.array_equal(got.reshape(-1).view(np.uint32).reshape(want.shape), want), (stop, t)
        assert mb.heap.check_invariants() == 0
        assert mb.heap.poll_error() == D.OK


@pytest.mark.parametrize("rec,n", [([4, 1], 4097), ([4, 4, 4], 3), ([4, 8, 4, 1], 5)])
def test_canonical_dump_odd_record_sizes(D, rec, n):
    """Record sizes that are not multiples of 8 (5, 12, 17 B) with odd live
    counts: the dump's cursor stays aligned and the records equal
    what the user kernel wrote."""
    heap = D.Heap([rec], 1 << 24)
    out = torch.zeros(n, dtype=torch.int64, device="cuda")
    heap.launch(D.K_LS_ALLOC, n, D.LsArgs(out.data_ptr(), 1, 0))
    torch.cuda.synchronize()
    recs = heap.canonical_dump(0)
    assert recs.shape == (n, sum(rec))
    assert heap.poll_error() == D.OK
