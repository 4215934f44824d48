"""Thin ctypes binding of libdsr.so (include/dsr.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  PyTorch is used
for device memory (the heap buffer is a torch uint8 CUDA tensor) and streams.

There is no CPU fallback: if libdsr.so cannot be loaded, or no CUDA device is
present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
import os as _os
# DSR_LIBPATH: an alternative build of the same library (A/B experiments only)
LIBPATH = Path(_os.environ["DSR_LIBPATH"]) if _os.environ.get("DSR_LIBPATH") else PKG / "libdsr.so"

MAX_TYPES, MAX_FIELDS, MAX_LEVELS = 8, 16, 6

# status codes
OK, ERR_INVALID, ERR_OOM, ERR_CUDA, ERR_RETRY_BUDGET, ERR_INVARIANT, ERR_UNSUPPORTED = range(7)
# flags
F_NO_ROTATE, F_NO_COALESCE, F_STATS, F_SPIN_ON_OOM, F_NO_HINT, F_CTA_NEW, F_HOME_ROT, F_SLOT_ROTATE = (
    0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40, 0x80)
F_SCALAR_DOALL = 0x100
F_QUAD_FREE = 0x200
F_BULK_DENSE = 0x400

# ids (mirror include/dsr.h)
K_MB_NEW, M_MB_REDUCE, M_MB_FREE_ODD, M_MB_FREE_ALL = 1, 1, 2, 3
K_MB_NEW_BULK = 8
K_LS_ALLOC, K_LS_FREE = 2, 3
K_REPLAY, K_TORTURE, M_COLLECT = 4, 5, 4
K_INH_NEW, K_INH_READ, M_INH_BUMP, M_INH_SUM, M_INH_SPAWN = 6, 7, 5, 6, 7
K_GOL_INIT_ALIVE, K_GOL_INIT_CAND, K_GOL_HALO_PACK, K_GOL_HALO_APPLY, K_GOL_HALO_PUSH = 10, 11, 12, 13, 14


def gol_peer_flags(W: int) -> int:
    """Byte offset of the two u32 flags in a peer-mode GoL halo (dsr.h DSR_GOL_PEER_FLAGS)."""
    return (6 * W + 15) & ~15


def gol_peer_halo_bytes(W: int) -> int:
    return gol_peer_flags(W) + 16
M_GOL_CAND_PREPARE, M_GOL_ALIVE_PREPARE, M_GOL_CAND_UPDATE, M_GOL_ALIVE_UPDATE, M_GOL_DUMP = 10, 11, 12, 13, 14
M_GOL_CAND_PREPARE_TILED, M_GOL_ALIVE_PREPARE_TILED, M_GOL_CAND_UPDATE_TILED, M_GOL_ALIVE_UPDATE_TILED = 15, 16, 17, 18
C_WT_CELL, K_WT_INIT_AGENTS = 20, 21
(K_WT_HALO_REQ_PACK, K_WT_HALO_REQ_APPLY, K_WT_HALO_GRANT_APPLY, K_WT_HALO_MIG_APPLY, K_WT_HALO_OCC_PACK,
 K_WT_HALO_OCC_APPLY) = range(22, 28)


def wt_halo_layout(W: int) -> dict:
    """Byte offsets of the Wa-Tor halo segments (dsr.h DSR_WT_HALO_*): name -> (out, in, bytes per side)."""
    mig_out = (12 * W + 15) & ~15
    return {"req": (0, 2 * W, W), "grant": (4 * W, 6 * W, W), "occ": (8 * W, 10 * W, W),
            "mig": (mig_out, mig_out + 24 * W, 12 * W), "bytes": mig_out + 48 * W}
(M_WT_CELL_PREPARE, M_WT_FISH_PREPARE, M_WT_CELL_DECIDE_FISH, M_WT_FISH_UPDATE, M_WT_SHARK_PREPARE,
 M_WT_CELL_DECIDE_SHARK, M_WT_SHARK_UPDATE, M_WT_DUMP) = range(20, 28)
C_NB_BODY, K_NB_CLEAR_SNAPSHOT, K_NB_CLAIM, K_NB_SIGNAL, K_NB_PUSH_TARGET = 30, 30, 31, 32, 33
(M_NB_SNAPSHOT, M_NB_FORCE, M_NB_MOVE, M_NB_PREPARE_MERGE, M_NB_CLAIM, M_NB_ABSORB, M_NB_DELETE_MERGED,
 M_NB_DUMP) = range(30, 38)


class TypeDesc(C.Structure):
    _fields_ = [("num_fields", C.c_uint32), ("field_bytes", C.c_uint32 * MAX_FIELDS), ("parent", C.c_uint32)]


class Layout(C.Structure):
    _fields_ = [
        ("ntypes", C.c_uint32), ("cap", C.c_uint32 * MAX_TYPES),
        ("col_off", (C.c_uint32 * MAX_FIELDS) * MAX_TYPES), ("block_bytes", C.c_uint32),
        ("M", C.c_uint64), ("nlevels", C.c_uint32), ("level_words", C.c_uint64 * 8),
        ("off_data", C.c_uint64), ("off_alloc_bm", C.c_uint64), ("off_iter_bm", C.c_uint64),
        ("off_type", C.c_uint64), ("off_R", C.c_uint64), ("off_bitmaps", C.c_uint64),
        ("bitmap_words", C.c_uint64), ("total_bytes", C.c_uint64),
    ]

    def to_dict(self):
        T = self.ntypes
        return {
            "cap": [self.cap[t] for t in range(T)],
            "col_off": [list(self.col_off[t]) for t in range(T)],
            "block_bytes": self.block_bytes, "M": self.M, "nlevels": self.nlevels,
            "level_words": [self.level_words[i] for i in range(self.nlevels)],
            "off_data": self.off_data, "off_alloc_bm": self.off_alloc_bm, "off_iter_bm": self.off_iter_bm,
            "off_type": self.off_type, "off_R": self.off_R, "off_bitmaps": self.off_bitmaps,
            "bitmap_words": self.bitmap_words, "total_bytes": self.total_bytes,
        }


class Config(C.Structure):
    _fields_ = [("active_retries", C.c_uint32), ("flags", C.c_uint32), ("seed", C.c_uint64),
                ("max_blocks", C.c_uint64)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("allocs", "frees", "block_inits", "block_frees", "rollbacks",
                                          "invalidate_fail", "reserve_retries", "oom", "requests", "finds",
                                          "find_fails", "reserve_zero", "cyc_find", "cyc_slow", "cyc_reserve",
                                          "cyc_request", "hint_zero")]

    def to_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


# ---- argument structs (mirror include/dsr.h)
class MbNewArgs(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("t0", C.c_uint64), ("in_", C.c_void_p), ("in_host", C.c_uint32),
                ("pad_", C.c_uint32)]


class MbReduceArgs(C.Structure):
    _fields_ = [("out3", C.c_void_p)]


class InhArgs(C.Structure):
    _fields_ = [("handles", C.c_void_p), ("ntypes", C.c_uint32), ("spawn_id0", C.c_uint32), ("out", C.c_void_p),
                ("vals", C.c_void_p)]


class LsArgs(C.Structure):
    _fields_ = [("handles", C.c_void_p), ("per_thread", C.c_uint32), ("type", C.c_uint32)]


class ReplayArgs(C.Structure):
    _fields_ = [("ops", C.c_void_p), ("nops", C.c_uint64), ("handles_out", C.c_void_p)]


class TortureArgs(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("iters", C.c_uint32), ("keep", C.c_uint32), ("ledger", C.c_void_p),
                ("errors", C.c_void_p)]


class CollectArgs(C.Structure):
    _fields_ = [("out", C.c_void_p), ("count", C.c_void_p)]


class GolArgs(C.Structure):
    _fields_ = [("cell", C.c_void_p), ("W", C.c_uint32), ("H", C.c_uint32), ("alive0", C.c_void_p),
                ("dump", C.c_void_p), ("ghost", C.c_uint32), ("halo", C.c_void_p), ("bits", C.c_void_p),
                ("peer_up", C.c_void_p), ("peer_down", C.c_void_p), ("gen", C.c_uint32)]


class WatorArgs(C.Structure):
    _fields_ = [("cells", C.c_void_p), ("W", C.c_uint32), ("H", C.c_uint32), ("FB", C.c_uint32),
                ("SB", C.c_uint32), ("SS", C.c_uint32), ("seed", C.c_uint64), ("step", C.c_uint32),
                ("kind0", C.c_void_p), ("egg0", C.c_void_p), ("energy0", C.c_void_p),
                ("out_kind", C.c_void_p), ("out_egg", C.c_void_p), ("out_energy", C.c_void_p),
                ("counters", C.c_void_p), ("ghost", C.c_uint32), ("y0", C.c_uint32), ("Hg", C.c_uint32),
                ("halo", C.c_void_p), ("step_dev", C.c_void_p)]


class NbodyStaticArgs(C.Structure):
    _fields_ = [("S", C.c_void_p), ("V", C.c_void_p), ("target", C.c_void_p), ("incoming", C.c_void_p),
                ("scratch", C.c_void_p), ("G", C.c_float), ("dt", C.c_float), ("eps", C.c_float), ("R", C.c_float),
                ("n", C.c_uint32), ("merges", C.c_uint32), ("live", C.c_void_p)]


class GolStaticArgs(C.Structure):
    _fields_ = [("W", C.c_uint32), ("H", C.c_uint32), ("cur", C.c_void_p), ("next", C.c_void_p)]


class WatorStaticArgs(C.Structure):
    _fields_ = [("W", C.c_uint32), ("H", C.c_uint32), ("FB", C.c_uint32), ("SB", C.c_uint32), ("SS", C.c_uint32),
                ("step", C.c_uint32), ("seed", C.c_uint64), ("kind", C.c_void_p), ("egg", C.c_void_p),
                ("energy", C.c_void_p), ("target", C.c_void_p), ("req", C.c_void_p), ("counters", C.c_void_p)]


class NbodyArgs(C.Structure):
    _fields_ = [("S", C.c_void_p), ("V", C.c_void_p), ("target", C.c_void_p), ("incoming", C.c_void_p),
                ("shandle", C.c_void_p),
                ("x0", C.c_void_p), ("y0", C.c_void_p), ("vx0", C.c_void_p), ("vy0", C.c_void_p),
                ("m0", C.c_void_p), ("G", C.c_float), ("dt", C.c_float), ("eps", C.c_float), ("R", C.c_float),
                ("n_total", C.c_uint32), ("id_lo", C.c_uint32), ("id_hi", C.c_uint32), ("out", C.c_void_p),
                ("scratch", C.c_void_p), ("live", C.c_void_p),
                ("npeers", C.c_uint32), ("rank", C.c_uint32), ("world", C.c_uint32), ("epoch", C.c_uint32),
                ("flags", C.c_void_p), ("peer_S", C.c_void_p * 7), ("peer_V", C.c_void_p * 7),
                ("peer_target", C.c_void_p * 7), ("peer_flags", C.c_void_p * 7)]


class DsrError(RuntimeError):
    def __init__(self, what, status):
        super().__init__(f"{what} failed: {status_str(status)}")
        self.status = status


_lib = None
vp = C.c_void_p


def lib():
    """Load libdsr.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not LIBPATH.exists():
            raise RuntimeError(f"{LIBPATH} is missing; run `python -m paper_1810_11765_b200.build` "
                               "(the CUDA extension is required, there is no CPU path)")
        L = C.CDLL(str(LIBPATH))
        st = C.c_int
        L.dsr_layout_compute.restype = st
        L.dsr_layout_compute.argtypes = [C.POINTER(TypeDesc), C.c_uint32, C.c_uint64, C.POINTER(Layout)]
        L.dsr_heap_create.restype = st
        L.dsr_heap_create.argtypes = [C.POINTER(TypeDesc), C.c_uint32, vp, C.c_uint64, C.POINTER(Config), vp,
                                      C.POINTER(vp)]
        L.dsr_heap_reset.restype = st
        L.dsr_heap_reset.argtypes = [vp, vp]
        L.dsr_heap_destroy.restype = st
        L.dsr_heap_destroy.argtypes = [vp]
        L.dsr_heap_layout.restype = st
        L.dsr_heap_layout.argtypes = [vp, C.POINTER(Layout)]
        L.dsr_heap_configure.restype = st
        L.dsr_heap_configure.argtypes = [vp, C.POINTER(Config)]
        if hasattr(L, "dsr_probe_atomics"):       # (absent in older builds loaded via DSR_LIBPATH for A/B runs)
            L.dsr_probe_atomics.restype = st
            L.dsr_probe_atomics.argtypes = [vp, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64), vp]
        L.dsr_ipc_handle.restype = st
        L.dsr_ipc_handle.argtypes = [vp, vp, C.POINTER(C.c_uint64)]
        L.dsr_ipc_open.restype = st
        L.dsr_ipc_open.argtypes = [vp, C.POINTER(vp)]
        L.dsr_ipc_close.restype = st
        L.dsr_ipc_close.argtypes = [vp]
        L.dsr_wator_static_step.restype = st
        L.dsr_wator_static_step.argtypes = [C.POINTER(WatorStaticArgs), C.c_uint32, vp]
        L.dsr_nbody_static_step.restype = st
        L.dsr_nbody_static_step.argtypes = [C.POINTER(NbodyStaticArgs), C.c_uint32, vp]
        L.dsr_gol_static_step.restype = st
        L.dsr_gol_static_step.argtypes = [C.POINTER(GolStaticArgs), C.c_uint32, vp]
        L.dsr_parallel_new.restype = st
        L.dsr_parallel_new.argtypes = [vp, C.c_uint32, C.c_uint64, C.c_uint32, vp, C.c_size_t, vp]
        L.dsr_parallel_do.restype = st
        L.dsr_parallel_do.argtypes = [vp, C.c_uint32, C.c_uint32, vp, C.c_size_t, vp]
        L.dsr_doall_prologue.restype = st
        L.dsr_doall_prologue.argtypes = [vp, C.c_uint32, C.c_uint32, vp]
        L.dsr_doall_body.restype = st
        L.dsr_doall_body.argtypes = [vp, C.c_uint32, C.c_uint32, vp, C.c_size_t, vp]
        L.dsr_reserve_blocks.restype = st
        L.dsr_reserve_blocks.argtypes = [vp, C.c_uint32, C.c_uint64, vp]
        L.dsr_trim.restype = st
        L.dsr_trim.argtypes = [vp, C.c_uint32, vp]
        L.dsr_launch.restype = st
        L.dsr_launch.argtypes = [vp, C.c_uint32, C.c_uint64, vp, C.c_size_t, vp]
        L.dsr_live_count.restype = st
        L.dsr_live_count.argtypes = [vp, C.c_uint32, vp, vp]
        L.dsr_live_count_sync.restype = st
        L.dsr_live_count_sync.argtypes = [vp, C.c_uint32, C.POINTER(C.c_uint64), vp]
        L.dsr_poll_error.restype = st
        L.dsr_poll_error.argtypes = [vp, vp]
        L.dsr_check_invariants.restype = st
        L.dsr_check_invariants.argtypes = [vp, vp, C.POINTER(C.c_uint64)]
        L.dsr_fragmentation.restype = st
        L.dsr_fragmentation.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_uint64), vp]
        L.dsr_stats.restype = st
        L.dsr_stats.argtypes = [vp, C.POINTER(Counters), vp]
        L.dsr_stats_reset.restype = st
        L.dsr_stats_reset.argtypes = [vp, vp]
        L.dsr_copy_state.restype = st
        L.dsr_copy_state.argtypes = [vp, C.c_uint32, C.c_uint32, vp, C.c_size_t, C.POINTER(C.c_size_t), vp]
        L.dsr_canonical_dump.restype = st
        L.dsr_canonical_dump.argtypes = [vp, C.c_uint32, vp, C.c_size_t, C.POINTER(C.c_size_t), vp]
        L.dsr_device_view_bytes.restype = C.c_size_t
        L.dsr_device_view_bytes.argtypes = []
        L.dsr_device_view.restype = st
        L.dsr_device_view.argtypes = [vp, vp, C.c_size_t]
        L.dsr_kernel_launches.restype = C.c_uint64
        L.dsr_kernel_launches.argtypes = []
        L.dsr_status_str.restype = C.c_char_p
        L.dsr_status_str.argtypes = [st]
        L.dsr_build_info.restype = C.c_char_p
        L.dsr_build_info.argtypes = []
        _lib = L
    return _lib


def status_str(s: int) -> str:
    return lib().dsr_status_str(s).decode()


def check(what: str, s: int):
    if s != OK:
        raise DsrError(what, s)


def kernel_launches() -> int:
    return lib().dsr_kernel_launches()


def type_descs(type_fields, parents=None):
    """parents[t]: index of t's base type, or None / -1 (no base)."""
    arr = (TypeDesc * len(type_fields))()
    for t, fields in enumerate(type_fields):
        if not 1 <= len(fields) <= MAX_FIELDS:
            raise ValueError("1..16 fields per type")
        arr[t].num_fields = len(fields)
        for f, b in enumerate(fields):
            arr[t].field_bytes[f] = b
        p = parents[t] if parents is not None else None
        arr[t].parent = 0 if p is None or p < 0 else p + 1
    return arr


def layout_compute(type_fields, heap_bytes, parents=None) -> dict:
    L = Layout()
    check("dsr_layout_compute", lib().dsr_layout_compute(type_descs(type_fields, parents), len(type_fields),
                                                          heap_bytes, C.byref(L)))
    return L.to_dict()


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _args(a):
    if a is None:
        return None, 0
    return C.byref(a), C.sizeof(a)


class Heap:
    """A DynaSOAr heap in a torch-owned device buffer (the host handle
    allocates one large buffer on the GPU)."""

    def __init__(self, type_fields, heap_bytes, device=None, retries=5, flags=0, seed=0x5EED, stream=None,
                 parents=None, max_blocks=0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the DynaSOAr hot path runs only on the GPU")
        self.type_fields = [list(f) for f in type_fields]
        self.ntypes = len(type_fields)
        self.device = torch.device(device or "cuda")
        self.buf = torch.empty(heap_bytes, dtype=torch.uint8, device=self.device)
        self.cfg = Config(retries, flags, seed, max_blocks)
        self.stream = stream
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check("dsr_heap_create", lib().dsr_heap_create(type_descs(type_fields, parents), self.ntypes,
                                                           C.c_void_p(self.buf.data_ptr()), heap_bytes,
                                                           C.byref(self.cfg), self._s(), C.byref(h)))
        self.h = h
        L = Layout()
        check("dsr_heap_layout", lib().dsr_heap_layout(self.h, C.byref(L)))
        self.layout = L.to_dict()
        self.M = self.layout["M"]
        self.cap = self.layout["cap"]

    def _s(self, stream=None):
        return _stream_ptr(stream if stream is not None else self.stream)

    def close(self):
        if getattr(self, "h", None):
            lib().dsr_heap_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def configure(self, retries=None, flags=None, seed=None):
        if retries is not None:
            self.cfg.active_retries = retries
        if flags is not None:
            self.cfg.flags = flags
        if seed is not None:
            self.cfg.seed = seed
        check("dsr_heap_configure", lib().dsr_heap_configure(self.h, C.byref(self.cfg)))

    def reset(self, stream=None):
        check("dsr_heap_reset", lib().dsr_heap_reset(self.h, self._s(stream)))

    def parallel_new(self, type_, n, ctor_id, args=None, stream=None):
        p, nb = _args(args)
        check("dsr_parallel_new", lib().dsr_parallel_new(self.h, type_, n, ctor_id, p, nb, self._s(stream)))

    def parallel_do(self, type_, method_id, args=None, stream=None):
        p, nb = _args(args)
        check("dsr_parallel_do", lib().dsr_parallel_do(self.h, type_, method_id, p, nb, self._s(stream)))

    def doall_prologue(self, type_, method_id, stream=None):
        check("dsr_doall_prologue", lib().dsr_doall_prologue(self.h, type_, method_id, self._s(stream)))

    def doall_body(self, type_, method_id, args=None, stream=None):
        p, nb = _args(args)
        check("dsr_doall_body", lib().dsr_doall_body(self.h, type_, method_id, p, nb, self._s(stream)))

    def reserve_blocks(self, type_, nblocks, stream=None):
        check("dsr_reserve_blocks", lib().dsr_reserve_blocks(self.h, type_, nblocks, self._s(stream)))

    def trim(self, type_, stream=None):
        check("dsr_trim", lib().dsr_trim(self.h, type_, self._s(stream)))

    def launch(self, kernel_id, n, args, stream=None):
        p, nb = _args(args)
        check("dsr_launch", lib().dsr_launch(self.h, kernel_id, n, p, nb, self._s(stream)))

    def live_count_async(self, type_, dev_out, stream=None):
        check("dsr_live_count", lib().dsr_live_count(self.h, type_, C.c_void_p(dev_out.data_ptr()),
                                                     self._s(stream)))

    def live_count(self, type_, stream=None) -> int:
        v = C.c_uint64()
        check("dsr_live_count_sync", lib().dsr_live_count_sync(self.h, type_, C.byref(v), self._s(stream)))
        return v.value

    def poll_error(self, stream=None) -> int:
        return lib().dsr_poll_error(self.h, self._s(stream))

    def check_invariants(self, stream=None) -> int:
        f = C.c_uint64()
        s = lib().dsr_check_invariants(self.h, self._s(stream), C.byref(f))
        if s not in (OK, ERR_INVARIANT):
            check("dsr_check_invariants", s)
        return f.value

    def fragmentation(self, stream=None):
        v = C.c_double()
        blocks = (C.c_uint64 * MAX_TYPES)()
        check("dsr_fragmentation", lib().dsr_fragmentation(self.h, C.byref(v), blocks, self._s(stream)))
        return v.value, [blocks[t] for t in range(self.ntypes)]

    def stats(self, stream=None) -> dict:
        c = Counters()
        check("dsr_stats", lib().dsr_stats(self.h, C.byref(c), self._s(stream)))
        return c.to_dict()

    def stats_reset(self, stream=None):
        check("dsr_stats_reset", lib().dsr_stats_reset(self.h, self._s(stream)))

    def canonical_dump(self, type_, stream=None):
        """Live objects of type_ as packed records (fields in declaration order,
        no padding), sorted by their bytes: (live, record_bytes) uint8 array."""
        import numpy as np
        used = C.c_size_t()
        rc = lib().dsr_canonical_dump(self.h, type_, None, 0, C.byref(used), self._s(stream))
        if rc not in (OK, ERR_INVALID):
            check("dsr_canonical_dump", rc)
        rb = sum(self.type_fields[type_])
        out = np.zeros(max(used.value, 1), dtype=np.uint8)
        check("dsr_canonical_dump", lib().dsr_canonical_dump(self.h, type_, out.ctypes.data, out.nbytes,
                                                             C.byref(used), self._s(stream)))
        return out[:used.value].reshape(-1, rb)

    def device_view(self) -> bytes:
        """The device heap descriptor (POD) for user kernels built against csrc/dsr_device.cuh."""
        n = lib().dsr_device_view_bytes()
        buf = (C.c_uint8 * n)()
        check("dsr_device_view", lib().dsr_device_view(self.h, buf, n))
        return bytes(buf)

    def copy_state(self, what, type_=0, stream=None):
        import numpy as np
        L = self.layout
        lw = sum(L["level_words"])
        nbytes = {0: 8 * self.M, 1: self.M, 2: 8 * lw, 3: 8 * lw, 4: 8 * lw, 5: 4 * self.M + 8}[what]
        out = np.zeros(nbytes, dtype=np.uint8)
        used = C.c_size_t()
        check("dsr_copy_state", lib().dsr_copy_state(self.h, what, type_, out.ctypes.data, nbytes, C.byref(used),
                                                     self._s(stream)))
        if what == 0:
            return out.view(np.uint64)
        if what == 1:
            return out
        if what == 5:
            cnt = int(out[4 * self.M:].view(np.uint64)[0])
            return out[:4 * self.M].view(np.uint32)[:cnt]
        words = out.view(np.uint64)
        levels, o = [], 0
        for n in L["level_words"]:
            levels.append(words[o:o + n])
            o += n
        return levels


def probe_atomics(buf, mode=0, iters=64, stream=None) -> int:
    """Launch the atomic-throughput probe on the torch CUDA tensor `buf`
    (dsr_probe_atomics); returns the number of atomics issued."""
    n = C.c_uint64(0)
    check("dsr_probe_atomics", lib().dsr_probe_atomics(C.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size(),
                                                       mode, iters, C.byref(n), _stream_ptr(stream)))
    return n.value



def ipc_handle(tensor):
    """(64-byte CUDA IPC handle of the allocation holding a torch CUDA tensor,
    the tensor's byte offset in it) -- dsr_ipc_handle."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64(0)
    check("dsr_ipc_handle", lib().dsr_ipc_handle(C.c_void_p(tensor.data_ptr()), buf, C.byref(off)))
    return buf.raw, off.value


def ipc_open(handle: bytes) -> int:
    """Device pointer of (the base of) another process's allocation (dsr_ipc_open)."""
    p = C.c_void_p()
    check("dsr_ipc_open", lib().dsr_ipc_open(C.create_string_buffer(bytes(handle), 64), C.byref(p)))
    return p.value


def ipc_close(ptr: int) -> None:
    check("dsr_ipc_close", lib().dsr_ipc_close(C.c_void_p(ptr)))


# ---------------------------------------------------------------- stream helpers for the host-side halo copies
def on_stream(stream):
    """Context: make `stream` (None = the current stream) torch's current
    stream, so torch copies / NCCL calls are ordered with the library's
    launches on it."""
    import torch
    return torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream())


class StreamJoin:
    """Context for device copies between several shards' streams (one-GPU
    loopback exchanges): the copies run on the first stream after it waited for
    all others, and every other stream waits for the copies afterwards."""

    def __init__(self, streams):
        import torch
        cur = torch.cuda.current_stream()
        self.streams = [s if s is not None else cur for s in streams]
        self.ctx = None

    def __enter__(self):
        import torch
        s0 = self.streams[0]
        for s in self.streams[1:]:
            if s != s0:
                s0.wait_stream(s)
        self.ctx = torch.cuda.stream(s0)
        return self.ctx.__enter__()

    def __exit__(self, *exc):
        r = self.ctx.__exit__(*exc)
        s0 = self.streams[0]
        for s in self.streams[1:]:
            if s != s0:
                s.wait_stream(s0)
        return r
