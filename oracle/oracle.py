"""ctypes wrapper of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_1810_11765_b200) never imports it; the CUDA path shares no code with
it.  See oracle/oracle.h for the passages each function follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
SOURCES = ["rng_layout.c", "hbitmap.c", "heapmodel.c", "microbench.c", "gol.c", "wator.c", "nbody.c"]

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> Path:
    """Compile the oracle with gcc (plain C, -ffp-contract=off)."""
    srcs = [HERE / s for s in SOURCES] + [HERE / "oracle.h", HERE / "store.h"]
    if not force and LIB.exists() and all(LIB.stat().st_mtime >= s.stat().st_mtime for s in srcs):
        return LIB
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", "-Wall", "-Wno-unused-function",
           "-o", str(LIB)] + [str(HERE / s) for s in SOURCES] + ["-lm"]
    subprocess.run(cmd, check=True)
    return LIB


class Layout(C.Structure):
    _fields_ = [
        ("ntypes", C.c_uint32),
        ("nfields", C.c_uint32 * 8),
        ("fsize", (C.c_uint32 * 16) * 8),
        ("cap", C.c_uint32 * 8),
        ("col_off", (C.c_uint32 * 16) * 8),
        ("block_bytes", C.c_uint32),
        ("M", C.c_uint64),
        ("nlevels", C.c_uint32),
        ("level_words", C.c_uint64 * 8),
    ]


class WatorParams(C.Structure):
    _fields_ = [("FB", C.c_uint32), ("SB", C.c_uint32), ("SS", C.c_uint32), ("seed", C.c_uint64)]


class NbodyParams(C.Structure):
    _fields_ = [("G", C.c_double), ("dt", C.c_double), ("eps", C.c_double), ("R", C.c_double),
                ("merges", C.c_int)]


_lib = None
HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_uint32, C.c_uint64)
HOOK_FOUND, HOOK_EMPTIED, HOOK_INVALIDATED = 0, 1, 2


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(str(build()))
        L.or_sm.restype = C.c_uint64
        L.or_sm.argtypes = [C.c_uint64]
        L.or_key.restype = C.c_uint64
        L.or_key.argtypes = [C.c_uint64] * 4
        L.or_layout.restype = C.c_int
        L.or_layout.argtypes = [C.c_uint32, u32p, u32p, C.c_uint64, C.POINTER(Layout)]
        vp = C.c_void_p
        L.or_bm_new.restype = vp
        L.or_bm_new.argtypes = [C.c_uint64, C.c_uint32, C.c_int]
        L.or_bm_free.argtypes = [vp]
        for fn in ("or_bm_try_set", "or_bm_try_clear"):
            getattr(L, fn).restype = C.c_int
            getattr(L, fn).argtypes = [vp, C.c_uint32, C.c_uint64]
        for fn in ("or_bm_set", "or_bm_clear"):
            getattr(L, fn).restype = None
            getattr(L, fn).argtypes = [vp, C.c_uint32, C.c_uint64]
        L.or_bm_try_find_set.restype = C.c_int64
        L.or_bm_try_find_set.argtypes = [vp, C.c_uint32]
        L.or_bm_clear_any.restype = C.c_int64
        L.or_bm_clear_any.argtypes = [vp]
        L.or_bm_get.restype = C.c_int
        L.or_bm_get.argtypes = [vp, C.c_uint64]
        L.or_bm_indices.restype = C.c_uint64
        L.or_bm_indices.argtypes = [vp, C.c_uint32, u64p]
        L.or_bm_consistent.restype = C.c_int
        L.or_bm_consistent.argtypes = [vp]
        L.or_bm_word.restype = C.c_uint64
        L.or_bm_word.argtypes = [vp, C.c_uint32, C.c_uint64]
        L.or_bm_nlevels.restype = C.c_uint32
        L.or_bm_nlevels.argtypes = [vp]
        L.or_bm_level_words.restype = C.c_uint64
        L.or_bm_level_words.argtypes = [vp, C.c_uint32]
        L.or_bm_trace.argtypes = [vp, C.c_int]
        L.or_bm_ntrace.restype = C.c_uint32
        L.or_bm_ntrace.argtypes = [vp]
        L.or_bm_trace_get.argtypes = [vp, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_uint32)]
        L.or_bm_error.restype = C.c_int
        L.or_bm_error.argtypes = [vp]
        L.or_heap_new.restype = vp
        L.or_heap_new.argtypes = [C.c_uint32, u32p, u32p, C.c_uint64]
        L.or_heap_free.argtypes = [vp]
        L.or_heap_alloc.restype = C.c_uint64
        L.or_heap_alloc.argtypes = [vp, C.c_uint32]
        L.or_heap_dealloc.restype = C.c_int
        L.or_heap_dealloc.argtypes = [vp, C.c_uint64]
        L.or_heap_M.restype = C.c_uint64
        L.or_heap_M.argtypes = [vp]
        L.or_heap_alloc_bm.restype = C.c_uint64
        L.or_heap_alloc_bm.argtypes = [vp, C.c_uint64]
        L.or_heap_type.restype = C.c_uint32
        L.or_heap_type.argtypes = [vp, C.c_uint64]
        L.or_heap_bitmap.restype = vp
        L.or_heap_bitmap.argtypes = [vp, C.c_uint32, C.c_uint32]
        L.or_heap_live.restype = C.c_uint64
        L.or_heap_live.argtypes = [vp, C.c_uint32]
        L.or_heap_fragmentation.restype = C.c_double
        L.or_heap_fragmentation.argtypes = [vp]
        L.or_heap_error.restype = C.c_int
        L.or_heap_error.argtypes = [vp]
        L.or_heap_set_hook.argtypes = [vp, HOOK, vp, C.c_uint32]
        L.or_heap_counter.restype = C.c_uint64
        L.or_heap_counter.argtypes = [vp, C.c_uint32]
        L.or_handle_encode.restype = C.c_uint64
        L.or_handle_encode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32]
        L.or_handle_decode.argtypes = [C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.or_assign_num_blocks.restype = C.c_uint64
        L.or_assign_num_blocks.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64]
        L.or_assign_block_pos.restype = C.c_uint64
        L.or_assign_block_pos.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_assign_slot.restype = C.c_uint32
        L.or_assign_slot.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_microbench.restype = C.c_int
        L.or_microbench.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p]
        L.or_microbench_live.restype = C.c_int
        L.or_microbench_live.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, u32p,
                                         C.c_uint64, u64p]
        L.or_gol_run.restype = C.c_int
        L.or_gol_run.argtypes = [C.c_uint32, C.c_uint32, u8p, C.c_uint32, C.c_uint64, vp, C.c_uint64, vp]
        L.or_life_dense.restype = None
        L.or_life_dense.argtypes = [C.c_uint32, C.c_uint32, u8p, C.c_uint32]
        L.or_wator_run.restype = C.c_int
        L.or_wator_run.argtypes = [C.c_uint32, C.c_uint32, u8p, u32p, u32p, C.POINTER(WatorParams),
                                   C.c_uint32, C.c_uint32, C.c_uint64, vp]
        L.or_wator_dense.restype = C.c_int
        L.or_wator_dense.argtypes = [C.c_uint32, C.c_uint32, u8p, u32p, u32p, C.POINTER(WatorParams),
                                     C.c_uint32, C.c_uint32, vp]
        L.or_nbody_run.restype = C.c_int
        L.or_nbody_run.argtypes = [C.c_uint32, f32p, f32p, f32p, f32p, f32p, u8p, C.POINTER(NbodyParams),
                                   C.c_uint32]
        _lib = L
    return _lib


# ---------------------------------------------------------------- helpers
def sm(x: int) -> int:
    return lib().or_sm(x)


def key(seed: int, step: int, phase: int, idx: int) -> int:
    return lib().or_key(seed, step, phase, idx)


def _flat(type_fields):
    nf = np.array([len(f) for f in type_fields], dtype=np.uint32)
    fs = np.array([s for f in type_fields for s in f], dtype=np.uint32)
    return nf, fs


def layout(type_fields, heap_bytes):
    """type_fields: list of lists of field byte sizes.  Returns a dict: cap,
    col_off, block_bytes, M (the paper-derived bound on the block count of a
    heap of heap_bytes, see or_layout), nlevels, level_words (of M bits)."""
    nf, fs = _flat(type_fields)
    L = Layout()
    rc = lib().or_layout(len(type_fields), nf, fs, heap_bytes, C.byref(L))
    if rc != 0:
        raise ValueError(f"or_layout rc={rc}")
    T = len(type_fields)
    return {
        "cap": [L.cap[t] for t in range(T)],
        "col_off": [[L.col_off[t][f] for f in range(len(type_fields[t]))] for t in range(T)],
        "block_bytes": L.block_bytes,
        "M": L.M,
        "nlevels": L.nlevels,
        "level_words": [L.level_words[i] for i in range(L.nlevels)],
    }


class Bitmap:
    """O2 hierarchical bitmap with container width W (sequential)."""

    def __init__(self, n, W=64, all_set=False):
        self.p = lib().or_bm_new(n, W, 1 if all_set else 0)
        if not self.p:
            raise ValueError("bad bitmap")
        self.n, self.W = n, W

    def __del__(self):
        if getattr(self, "p", None):
            lib().or_bm_free(self.p)
            self.p = None

    def try_set(self, pos, level=0): return bool(lib().or_bm_try_set(self.p, level, pos))
    def try_clear(self, pos, level=0): return bool(lib().or_bm_try_clear(self.p, level, pos))
    def set(self, pos, level=0): lib().or_bm_set(self.p, level, pos)
    def clear(self, pos, level=0): lib().or_bm_clear(self.p, level, pos)
    def try_find_set(self): return lib().or_bm_try_find_set(self.p, 0)
    def clear_any(self): return lib().or_bm_clear_any(self.p)
    def get(self, pos): return bool(lib().or_bm_get(self.p, pos))
    def consistent(self): return bool(lib().or_bm_consistent(self.p))
    def error(self): return lib().or_bm_error(self.p)
    def nlevels(self): return lib().or_bm_nlevels(self.p)

    def indices(self):
        out = np.zeros(self.n + 1, dtype=np.uint64)
        k = lib().or_bm_indices(self.p, 0, out)
        return out[:k].copy()

    def words(self, level):
        nw = lib().or_bm_level_words(self.p, level)
        return np.array([lib().or_bm_word(self.p, level, i) for i in range(nw)], dtype=np.uint64)

    def trace(self, on=True): lib().or_bm_trace(self.p, 1 if on else 0)

    def trace_get(self):
        out = []
        for i in range(lib().or_bm_ntrace(self.p)):
            a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
            lib().or_bm_trace_get(self.p, i, C.byref(a), C.byref(b), C.byref(c))
            out.append((a.value, b.value, "set" if c.value else "clear"))
        return out


class _BorrowedBitmap(Bitmap):
    def __init__(self, p, n):
        self.p, self.n, self.W = p, n, 64

    def __del__(self):
        pass


class PaperHeap:
    """O2 sequential model of the paper's allocator (Algs. 1-9)."""

    def __init__(self, type_fields, M):
        """A heap of exactly M blocks for the given types."""
        nf, fs = _flat(type_fields)
        self.p = lib().or_heap_new(len(type_fields), nf, fs, M)
        if not self.p:
            raise ValueError("bad heap")
        self.ntypes = len(type_fields)
        self.M = lib().or_heap_M(self.p)

    def __del__(self):
        if getattr(self, "p", None):
            lib().or_heap_free(self.p)
            self.p = None

    def on(self, point, fn):
        """Arm a one-shot hook at `point` (HOOK_*): fn(bid) runs "another
        thread's" operations on this heap at that linearisation point."""
        if not hasattr(self, "_fns"):
            self._fns = {}
            self._cb = HOOK(lambda ctx, pt, bid: self._fns[pt](bid))   # kept alive with the heap
        self._fns[point] = fn
        lib().or_heap_set_hook(self.p, self._cb, None, point)

    def counters(self):
        return {k: lib().or_heap_counter(self.p, i)
                for i, k in enumerate(["rollbacks", "invalidate_fail", "invalidate_retry", "deferred_deactivation"])}

    def alloc(self, t): return lib().or_heap_alloc(self.p, t)
    def dealloc(self, h): return lib().or_heap_dealloc(self.p, h)
    def alloc_bm(self, b): return lib().or_heap_alloc_bm(self.p, b)
    def type(self, b): return lib().or_heap_type(self.p, b)
    def live(self, t): return lib().or_heap_live(self.p, t)
    def fragmentation(self): return lib().or_heap_fragmentation(self.p)
    def error(self): return lib().or_heap_error(self.p)

    def bitmap(self, which, t=0):
        return _BorrowedBitmap(lib().or_heap_bitmap(self.p, which, t), self.M)

    def alloc_bm_array(self):
        return np.array([self.alloc_bm(b) for b in range(self.M)], dtype=np.uint64)

    def type_array(self):
        return np.array([self.type(b) for b in range(self.M)], dtype=np.uint8)


def handle_encode(t, cap, bid, slot):
    return lib().or_handle_encode(t, cap, bid, slot)


def handle_decode(h):
    a, b, c, d = C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_uint32()
    lib().or_handle_decode(h, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
    return a.value, b.value, c.value, d.value


def assign_num_blocks(r, NT, n, tid): return lib().or_assign_num_blocks(r, NT, n, tid)
def assign_block_pos(NT, n, tid, k): return lib().or_assign_block_pos(NT, n, tid, k)
def assign_slot(NT, n, tid, k): return lib().or_assign_slot(NT, n, tid, k)


def microbench(seed, n1, n2, order_seed=0):
    out = np.zeros(18, dtype=np.uint64)
    live = np.zeros(18, dtype=np.uint64)
    rc = lib().or_microbench(seed, n1, n2, order_seed, out, live)
    if rc:
        raise RuntimeError(f"or_microbench rc={rc}")
    return out.reshape(2, 3, 3), live.reshape(6, 3)


def microbench_live(seed, n1, n2, stop, ty):
    """Canonical dump of type ty's live objects after phase `stop` (1, 3 or 4):
    (live, nfields) uint32 records sorted by their little-endian bytes (the
    order of dsr_canonical_dump)."""
    nf = [3, 4, 6][ty]
    cnt = np.zeros(1, dtype=np.uint64)
    lib().or_microbench_live(seed, n1, n2, stop, ty, np.zeros(1, dtype=np.uint32), 0, cnt)
    k = int(cnt[0])
    out = np.zeros(max(k, 1) * nf, dtype=np.uint32)
    rc = lib().or_microbench_live(seed, n1, n2, stop, ty, out, out.size, cnt)
    if rc:
        raise RuntimeError(f"or_microbench_live rc={rc}")
    return sort_records(out[:k * nf].reshape(k, nf))


def sort_records(recs):
    """Rows of a (k, n) little-endian array sorted lexicographically by their bytes."""
    recs = np.ascontiguousarray(recs)
    b = recs.view(np.uint8).reshape(len(recs), -1)
    order = np.lexsort(b.T[::-1]) if len(recs) else np.zeros(0, dtype=np.int64)
    return recs[order]


def gol_run(alive, gens, order_seed=0, dump=False):
    """alive: (H, W) uint8.  Returns (alive_after, [per-gen (n,4) u32 records] or None)."""
    H, W = alive.shape
    a = np.ascontiguousarray(alive, dtype=np.uint8).reshape(-1).copy()
    if dump:
        cap = W * H * max(gens, 1)
        buf = np.zeros(4 * cap, dtype=np.uint32)
        counts = np.zeros(max(gens, 1), dtype=np.uint64)
        rc = lib().or_gol_run(W, H, a, gens, order_seed, buf.ctypes.data, cap, counts.ctypes.data)
        if rc:
            raise RuntimeError(f"or_gol_run rc={rc}")
        recs, off = [], 0
        for g in range(gens):
            k = int(counts[g])
            recs.append(buf[4 * off: 4 * (off + k)].reshape(k, 4).copy())
            off += k
        return a.reshape(H, W), recs
    rc = lib().or_gol_run(W, H, a, gens, order_seed, None, 0, None)
    if rc:
        raise RuntimeError(f"or_gol_run rc={rc}")
    return a.reshape(H, W), None


def life_dense(alive, gens):
    H, W = alive.shape
    a = np.ascontiguousarray(alive, dtype=np.uint8).reshape(-1).copy()
    lib().or_life_dense(W, H, a, gens)
    return a.reshape(H, W)


def wator_run(kind, egg, energy, FB, SB, SS, seed, steps, step0=0, order_seed=0, dense=False):
    """kind/egg/energy: (H, W) arrays.  Returns (kind, egg, energy, counters[steps, 6])."""
    H, W = kind.shape
    k = np.ascontiguousarray(kind, dtype=np.uint8).reshape(-1).copy()
    e = np.ascontiguousarray(egg, dtype=np.uint32).reshape(-1).copy()
    en = np.ascontiguousarray(energy, dtype=np.uint32).reshape(-1).copy()
    cnt = np.zeros(6 * max(steps, 1), dtype=np.uint64)
    p = WatorParams(FB, SB, SS, seed)
    if dense:
        rc = lib().or_wator_dense(W, H, k, e, en, C.byref(p), step0, steps, cnt.ctypes.data)
    else:
        rc = lib().or_wator_run(W, H, k, e, en, C.byref(p), step0, steps, order_seed, cnt.ctypes.data)
    if rc:
        raise RuntimeError(f"wator rc={rc}")
    return k.reshape(H, W), e.reshape(H, W), en.reshape(H, W), cnt.reshape(-1, 6)[:steps]


def nbody_run(state, G, dt, eps, R, merges, steps):
    """state: dict of x, y, vx, vy, m (float32) and alive (uint8); copied, returned updated."""
    s = {k: np.ascontiguousarray(v).copy() for k, v in state.items()}
    p = NbodyParams(G, dt, eps, R, 1 if merges else 0)
    n = len(s["x"])
    rc = lib().or_nbody_run(n, s["x"], s["y"], s["vx"], s["vy"], s["m"], s["alive"], C.byref(p), steps)
    if rc:
        raise RuntimeError(f"nbody rc={rc}")
    return s
