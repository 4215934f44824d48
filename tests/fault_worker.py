"""Worker for tests/test_gpu_debug_fault.py: runs in a subprocess with
DSR_LIBPATH pointing at a debug / fault-injection build of libdsr.so (one
library per process), prints one JSON line of results."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np
import torch

from paper_1810_11765_b200 import dsr


def torture(seed, nthreads, iters, max_blocks, bulk_check):
    """Divergent new/destroy on a tiny heap (blocks re-typed all the time),
    then the ledger / live-set / invariant checks of test_gpu_allocator."""
    tf = [[4, 4, 4], [4, 4, 4, 4], [4] * 6, [4] * 16, [4, 4]]
    heap = dsr.Heap(tf, 1 << 24, flags=dsr.F_STATS, max_blocks=max_blocks)
    ledger = torch.zeros(nthreads * 8, dtype=torch.int64, device="cuda")
    errors = torch.zeros(1, dtype=torch.int64, device="cuda")
    heap.launch(dsr.K_TORTURE, nthreads, dsr.TortureArgs(seed, iters, 1, ledger.data_ptr(), errors.data_ptr()))
    torch.cuda.synchronize()
    out = {"canary_errors": int(errors.item()), "poll": heap.poll_error(), "M": heap.M}
    out["audit_failures"] = heap.check_invariants()
    led = ledger.cpu().numpy().view(np.uint64)
    led = np.sort(led[led != 0])
    got = []
    for t in range(len(tf)):
        o = torch.zeros(len(led) + 1, dtype=torch.int64, device="cuda")
        c = torch.zeros(1, dtype=torch.int64, device="cuda")
        heap.parallel_do(t, dsr.M_COLLECT, dsr.CollectArgs(o.data_ptr(), c.data_ptr()))
        torch.cuda.synchronize()
        got.append(o[:int(c.item())].cpu().numpy().view(np.uint64))
    got = np.sort(np.concatenate(got))
    out["ledger_unique"] = bool(len(np.unique(led)) == len(led))
    out["live_equals_ledger"] = bool(np.array_equal(got, led))
    st = heap.stats()
    out["stats"] = {k: int(st[k]) for k in ("allocs", "frees", "block_inits", "block_frees", "rollbacks",
                                            "invalidate_fail", "oom")}
    out["allocs_minus_frees_equals_live"] = int(st["allocs"] - st["frees"]) == len(led)
    for t in range(len(tf)):
        heap.parallel_do(t, dsr.M_MB_FREE_ALL)
    torch.cuda.synchronize()
    out["audit_after_drain"] = heap.check_invariants()
    out["live_after_drain"] = [heap.live_count(t) for t in range(len(tf))]
    out["poll_after_drain"] = heap.poll_error()
    if bulk_check:
        from oracle import oracle as O
        from paper_1810_11765_b200.microbench import Microbench
        mb = Microbench(n1=100_000, n2=50_000, seed=3, heap_bytes=16 << 20, flags=dsr.F_STATS)
        mb.step()
        torch.cuda.synchronize()
        out["bulk_microbench_equals_oracle"] = bool(np.array_equal(mb.results(), O.microbench(3, 100_000, 50_000)[0]))
        out["bulk_audit"] = mb.heap.check_invariants()
        out["bulk_poll"] = mb.heap.poll_error()
    return out


def double_destroy():
    """Destroying an object twice is illegal (Alg. 7 precondition).
    (a) the object's block still holds other objects: its bit is already 0
    when the second destroy's atomicAnd runs -- the debug build's precondition
    check reports it; (b) the whole block was freed in between: its bitmap is
    invalidated (all ones), so the precondition cannot see it, the second
    destroy "frees" a free block and its allocated.clear spins -- the
    debug build's spin bound reports it.  Both: DSR_ERR_RETRY_BUDGET."""
    out = {}
    heap = dsr.Heap([[4, 4]], 1 << 22, flags=dsr.F_STATS)
    hs = torch.zeros(64, dtype=torch.int64, device="cuda")
    heap.launch(dsr.K_LS_ALLOC, 64, dsr.LsArgs(hs.data_ptr(), 1, 0))
    one = hs[5:6].clone()
    heap.launch(dsr.K_LS_FREE, 1, dsr.LsArgs(one.data_ptr(), 1, 0))
    torch.cuda.synchronize()
    out["a_first"] = heap.poll_error()
    heap.launch(dsr.K_LS_FREE, 1, dsr.LsArgs(one.data_ptr(), 1, 0))
    torch.cuda.synchronize()
    out["a_second"] = heap.poll_error()
    out["a_live"] = heap.live_count(0)
    out["a_audit"] = heap.check_invariants()
    heap2 = dsr.Heap([[4, 4]], 1 << 22, flags=dsr.F_STATS)
    n = 100
    hs2 = torch.zeros(n, dtype=torch.int64, device="cuda")
    heap2.launch(dsr.K_LS_ALLOC, n, dsr.LsArgs(hs2.data_ptr(), 1, 0))
    heap2.launch(dsr.K_LS_FREE, n, dsr.LsArgs(hs2.data_ptr(), 1, 0))
    torch.cuda.synchronize()
    out["b_first"] = heap2.poll_error()
    out["b_stats_first"] = {k: int(v) for k, v in heap2.stats().items() if k in ("allocs", "frees", "block_inits",
                                                                                  "block_frees")}
    heap2.launch(dsr.K_LS_FREE, n, dsr.LsArgs(hs2.data_ptr(), 1, 0))      # the same handles again
    torch.cuda.synchronize()
    out["b_second"] = heap2.poll_error()
    return out


if __name__ == "__main__":
    what = sys.argv[1]
    res = {"build": dsr.lib().dsr_build_info().decode()}
    if what == "torture":
        res.update(torture(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6] == "1"))
    elif what == "double_destroy":
        res.update(double_destroy())
    print(json.dumps(res), flush=True)
