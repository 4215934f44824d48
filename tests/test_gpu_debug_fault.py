"""Rare-path verification on the GPU (VERDICT r01 'what's missing' #4):

* a fault-injection build (-DDSR_FAULT: random 0.5-8 us pauses at the
  linearisation points, csrc/dsr_device.cuh) on tiny heaps, so that the
  branches only concurrency reaches -- the type-change rollback (Alg. 1 l.14,
  P:397) and the failed invalidation with its rollback (Alg. 9 l.8-13,
  P:1055-1063) -- actually run, with every quiescent invariant, the canaries
  and the ledger = live set still holding afterwards (the oracle pins the same
  branches sequentially: tests/test_oracle_heap.py "scripted interleavings");
* the debug build (-DDSR_DEBUG): illegal use (a double destroy, Alg. 7's
  precondition P:1000) is reported as DSR_ERR_RETRY_BUDGET instead of
  corrupting or deadlocking the heap.
Each build is a separate library, loaded by tests/fault_worker.py in its own
process (DSR_LIBPATH)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def libs():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build
    return {"fault": build.build(variant="fault", defines=["DSR_DEBUG", "DSR_FAULT"]),
            "debug": build.build(variant="debug", defines=["DSR_DEBUG"])}


def run_worker(lib, *args, timeout=600):
    env = dict(os.environ, DSR_LIBPATH=str(lib))
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "fault_worker.py"), *map(str, args)], env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("seed,nthreads,iters,max_blocks", [(1, 8192, 60, 24), (2, 32768, 40, 96), (3, 4096, 200, 12)])
def test_fault_injection_reaches_rollbacks_and_stays_consistent(libs, seed, nthreads, iters, max_blocks):
    from paper_1810_11765_b200 import dsr
    r = run_worker(libs["fault"], "torture", seed, nthreads, iters, max_blocks, 1 if seed == 1 else 0)
    assert "fault" in r["build"] or "debug" in r["build"]
    assert r["M"] == max_blocks
    assert r["canary_errors"] == 0
    assert r["poll"] in (dsr.OK, dsr.ERR_OOM)                  # tiny heap: OOM is expected, no illegal use
    assert r["audit_failures"] == 0
    assert r["ledger_unique"] and r["live_equals_ledger"] and r["allocs_minus_frees_equals_live"]
    assert r["stats"]["rollbacks"] > 0, r["stats"]             # Alg. 1 l.14 ran
    assert r["stats"]["invalidate_fail"] > 0, r["stats"]       # Alg. 9 l.8 ran
    assert r["audit_after_drain"] == 0 and r["live_after_drain"] == [0] * 5
    assert r["poll_after_drain"] == dsr.OK
    if seed == 1:
        assert r["bulk_microbench_equals_oracle"] and r["bulk_audit"] == 0 and r["bulk_poll"] == dsr.OK


def test_debug_build_reports_double_destroy(libs):
    from paper_1810_11765_b200 import dsr
    r = run_worker(libs["debug"], "double_destroy")
    assert "debug" in r["build"]
    assert r["first_free"] == dsr.OK
    assert r["second_free"] == dsr.ERR_RETRY_BUDGET
    assert r["audit"] == 0 and r["live"] == 0
