"""User code outside the library and the canonical dump (SURVEY
c.8): a kernel compiled separately against csrc/dsr_device.cuh allocates and
destroys objects of a libdsr heap through dsr_device_view; the library's
host calls (live count, audit, canonical dump) see exactly those objects."""
import ctypes
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build, dsr
    build.build()
    return dsr


@pytest.fixture(scope="module")
def user_lib(D, tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    out = tmp_path_factory.mktemp("uk") / "libuser.so"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
           "-fPIC", "-I", str(ROOT / "paper_1810_11765_b200" / "csrc"), str(ROOT / "tests" / "user_kernel" /
                                                                          "user_objects.cu"), "-o", str(out)]
    subprocess.run(cmd, check=True, capture_output=True)
    lib = ctypes.CDLL(str(out))
    lib.user_launch.restype = ctypes.c_int
    lib.user_launch.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_void_p]
    return lib


def test_user_kernel_new_destroy_through_device_view(D, user_lib):
    n = 100_000
    heap = D.Heap([[4, 8]], 1 << 26)
    view = heap.device_view()
    handles = torch.zeros(n, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert user_lib.user_launch(view, len(view), n, handles.data_ptr(), 0, s) == 0
    torch.cuda.synchronize()
    assert heap.live_count(0) == n
    assert heap.check_invariants() == 0
    assert user_lib.user_launch(view, len(view), n, handles.data_ptr(), 1, s) == 0
    torch.cuda.synchronize()
    keep = np.array([i for i in range(n) if i % 3])
    assert heap.live_count(0) == len(keep)
    assert heap.check_invariants() == 0
    recs = heap.canonical_dump(0)                                   # (live, 12) packed {u32 id, u64 twice}
    ids = recs[:, :4].copy().view(np.uint32).ravel()
    twice = recs[:, 4:].copy().view(np.uint64).ravel()
    assert np.array_equal(np.sort(ids), keep.astype(np.uint32))
    assert np.array_equal(twice, 2 * ids.astype(np.uint64))
    assert all(bytes(recs[i]) <= bytes(recs[i + 1]) for i in range(0, len(recs) - 1, 997))   # sorted by bytes


def test_canonical_dump_wator_equals_oracle_state(D, O):
    """Placement-independent dump of Fish / Shark after 20 steps equals the
    records built from the oracle's dense state: Fish (cell, target = cell,
    egg), Shark (cell, target = cell, egg, energy)."""
    from paper_1810_11765_b200 import inputs as I, wator
    WT = dict(FB=6, SB=12, SS=6, seed=42)
    kind, egg, en = I.wator_init(80, 48, seed=3)
    sim = wator.WaTor(kind, egg, en, **WT)
    sim.run(20)
    k, e, g, _ = O.wator_run(kind, egg, en, steps=20, **WT)
    k, e, g = k.ravel(), e.ravel(), g.ravel()
    for T, kk, cols in ((wator.FISH, 1, 3), (wator.SHARK, 2, 4)):
        cells = np.nonzero(k == kk)[0].astype(np.uint32)
        fields = [cells, cells, e[cells].astype(np.uint32)] + ([g[cells].astype(np.uint32)] if cols == 4 else [])
        want = sorted(np.stack(fields, axis=1).astype("<u4").tobytes()[i * 4 * cols:(i + 1) * 4 * cols]
                      for i in range(len(cells)))
        got = sim.heap.canonical_dump(T)
        assert [bytes(r) for r in got] == want
