"""Allocator microbenchmark driver (BASELINE configs[4]; SURVEY c.4): the host
loop of dsr_launch / dsr_parallel_do calls.  All work runs in libdsr.so."""
from __future__ import annotations

import ctypes as C

from . import dsr

MB_TYPES = [[4, 4, 4], [4, 4, 4, 4], [4] * 6]   # A{3 x u32}, B{4 x u32}, C{6 x u32}
PHASES = ["init", "new1", "reduce2", "free3", "new4", "reduce5", "drain6"]


class Microbench:
    def __init__(self, n1=1 << 26, n2=1 << 25, seed=1, heap_bytes=None, device=None, retries=5, flags=0,
                 stream=None, reserve=False, reserve_slack=0.0, bulk=True):
        import torch
        self.n1, self.n2, self.seed = n1, n2, seed
        self.reserve = reserve      # dsr_reserve_blocks before / dsr_trim after the phase-1 burst (host foreknowledge; off by default)
        self.bulk = bulk            # K_MB_NEW_BULK (warp-cooperative requests, R-BULK) instead of per-thread K_MB_NEW
        self.kernel = dsr.K_MB_NEW_BULK if bulk else dsr.K_MB_NEW
        self.reserve_slack = reserve_slack   # extra fraction of blocks reserved (trimmed afterwards)
        if heap_bytes is None:
            # room for every object of phase 1 + 4 at the worst per-block fill, x2 for contention slack
            heap_bytes = max(64 << 20, int((n1 + n2) * 24 * 2.0))
        self.heap = dsr.Heap(MB_TYPES, heap_bytes, device=device, retries=retries, flags=flags, stream=stream)
        self.out = torch.zeros(18, dtype=torch.int64, device=self.heap.device)   # u64 bit patterns
        self.stream = stream

    @staticmethod
    def _counts(t0, n):
        """objects of A, B, C among threads t0 .. t0+n-1 ([A,A,B,C][t & 3])."""
        c = [0, 0, 0]
        for r in range(4):
            k = len(range((r - t0) % 4, n, 4))
            c[[0, 0, 1, 2][(t0 + (r - t0) % 4) & 3]] += k
        return c

    def _reduce_args(self, k):
        return dsr.MbReduceArgs(self.out.data_ptr() + 8 * k)

    def step(self, stream=None, events=None, body_events=None, inputs=None, before_new4=None, host_inputs=False,
             stop=None):
        """One pass of the whole hot path: heap init, new 2^26, reduce, free odd,
        new 2^25, reduce, drain.  `events`: optional list of 7 torch.cuda.Event
        pairs recorded around the phases; `body_events`: 6 pairs around the
        reduce bodies (k_mb_reduce) of phases 2 and 5 (timing only).  `inputs`:
        optional (in1, in2) device pointers to the field values of the phase-1 /
        phase-4 objects (inputs.mb_fields layout) instead of device-computed keys
        (host pointers with host_inputs=True: the library stages them, dsr.h);
        `before_new4`: called (host side) just before phase 4 is enqueued.
        `stop`: 1, 3 or 4 -- return after that phase (parity of the live set)."""
        h = self.heap
        s = stream if stream is not None else self.stream

        def ev(i, end):
            if events is not None:
                events[i][1 if end else 0].record(s)

        def reduce(t, k, j):
            h.doall_prologue(t, dsr.M_MB_REDUCE, s)
            if body_events is not None:
                body_events[j][0].record(s)
            h.doall_body(t, dsr.M_MB_REDUCE, self._reduce_args(k), s)
            if body_events is not None:
                body_events[j][1].record(s)

        ev(0, 0)
        h.reset(s)
        import torch
        with torch.cuda.stream(s if s is not None else torch.cuda.current_stream()):
            self.out.zero_()
        ev(0, 1)
        ev(1, 0)
        if self.reserve:
            # bulk slow path ahead of the burst: the blocks phase 1 needs
            for t, cnt in enumerate(self._counts(0, self.n1)):
                h.reserve_blocks(t, int(-(-cnt // self.heap.cap[t]) * (1.0 + self.reserve_slack)), s)
        in1, in2 = inputs if inputs is not None else (None, None)
        h.launch(self.kernel, self.n1, dsr.MbNewArgs(self.seed, 0, in1, int(bool(host_inputs))), s)
        if self.reserve:
            for t in range(3):
                h.trim(t, s)
        ev(1, 1)
        if stop == 1:
            return
        ev(2, 0)
        for t in range(3):
            reduce(t, 3 * t, t)
        ev(2, 1)
        ev(3, 0)
        for t in range(3):
            h.parallel_do(t, dsr.M_MB_FREE_ODD, None, s)
        ev(3, 1)
        if stop == 3:
            return
        if before_new4 is not None:
            before_new4()
        ev(4, 0); h.launch(self.kernel, self.n2, dsr.MbNewArgs(self.seed, self.n1, in2, int(bool(host_inputs))), s); ev(4, 1)
        if stop == 4:
            return
        ev(5, 0)
        for t in range(3):
            reduce(t, 9 + 3 * t, 3 + t)
        ev(5, 1)
        ev(6, 0)
        for t in range(3):
            h.parallel_do(t, dsr.M_MB_FREE_ALL, None, s)
        ev(6, 1)

    def results(self):
        """(2, 3, 3) numpy uint64: phase 2/5 x type x (count, sum, xor)."""
        import numpy as np
        return self.out.cpu().numpy().view(np.uint64).reshape(2, 3, 3)

    def counts(self):
        """Per-step operation counts for throughput metrics (needs results())."""
        r = self.results()
        ph2 = int(r[0, :, 0].sum())
        ph5 = int(r[1, :, 0].sum())
        freed3 = ph2 + self.n2 - ph5                 # phase 3 frees = phase-2 live + n2 - phase-5 live
        return {"allocs": self.n1 + self.n2, "frees": freed3 + ph5,
                "visits": ph2 + ph2 + ph5 + ph5,     # reduce2, free3, reduce5, drain6
                "scan_objects": ph2 + ph5}
