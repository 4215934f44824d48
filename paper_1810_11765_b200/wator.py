"""Wa-Tor driver: the host loop of eight dsr_parallel_do calls per step
(Table 1; reading R-WATOR).  BASELINE configs[1] (2048^2, 500 steps)."""
from __future__ import annotations

from . import dsr

WT_TYPES = [[4, 4, 4], [4, 4, 4, 4], [4, 8, 1, 1, 1, 1, 1]]   # Fish, Shark, Cell
FISH, SHARK, CELL = 0, 1, 2


def row_range(H: int, world: int, rank: int):
    """Rows owned by `rank` (contiguous bands; H % world == 0)."""
    if H % world:
        raise ValueError("H must be divisible by the number of shards")
    b = H // world
    return rank * b, (rank + 1) * b


class WaTor:
    """One heap for the whole torus, or -- with shard=(rank, P) -- one row band
    with two ghost rows.  Each half step then has four boundary
    exchanges (requests, grants, migrating agents, boundary occupancy); agents
    crossing a band boundary are destroyed by the sender and created by the
    owner of the arrival cell.  With P shards the result is the single-heap
    result bit for bit."""

    def __init__(self, kind, egg, energy, FB=6, SB=12, SS=6, seed=42, heap_bytes=None, device=None,
                 stream=None, retries=5, flags=0, step0=0, shard=None, exchange=None):
        import numpy as np
        import torch
        Hg, W = kind.shape
        self.shard, self.exchange, self.Hg = shard, exchange, Hg
        if shard is not None:
            r, P = shard
            y0, y1 = row_range(Hg, P, r)
            rows = [(y0 - 1) % Hg] + list(range(y0, y1)) + [y1 % Hg]
            kind, egg, energy = kind[rows], egg[rows], energy[rows]
            H, self.grid_rows, self.y0 = y1 - y0, y1 - y0 + 2, y0
        else:
            H, self.grid_rows, self.y0 = Hg, Hg, 0
        self.W, self.H, self.N = W, H, W * self.grid_rows
        if heap_bytes is None:
            heap_bytes = max(32 << 20, self.N * 96 + (16 << 20))
        self.heap = dsr.Heap(WT_TYPES, heap_bytes, device=device, retries=retries, flags=flags, stream=stream)
        dev = self.heap.device
        self.stream = stream
        self.cells = torch.zeros(self.N, dtype=torch.int64, device=dev)
        self.kind0 = torch.from_numpy(np.ascontiguousarray(kind, np.uint8).reshape(-1)).to(dev)
        self.egg0 = torch.from_numpy(np.ascontiguousarray(egg, np.uint32).reshape(-1).view(np.int32)).to(dev)
        self.energy0 = torch.from_numpy(np.ascontiguousarray(energy, np.uint32).reshape(-1).view(np.int32)).to(dev)
        self.out = torch.zeros(3, self.N, dtype=torch.int32, device=dev)
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)   # fish born, sharks born, eaten, starved
        self.halo_layout = dsr.wt_halo_layout(W)
        self.halo = torch.zeros(self.halo_layout["bytes"], dtype=torch.uint8, device=dev)
        self.args = dsr.WatorArgs(self.cells.data_ptr(), W, H, FB, SB, SS, seed, step0,
                                  self.kind0.data_ptr(), self.egg0.data_ptr(), self.energy0.data_ptr(),
                                  self.out[0].data_ptr(), self.out[1].data_ptr(), self.out[2].data_ptr(),
                                  self.counters.data_ptr(), 1 if shard is not None else 0, self.y0, Hg,
                                  self.halo.data_ptr() if shard is not None else None)
        self.heap.parallel_new(CELL, self.N, dsr.C_WT_CELL, self.args, stream)   # constructor i -> id i
        self.heap.launch(dsr.K_WT_INIT_AGENTS, self.N, self.args, stream)
        self.step_no = step0

    def stages(self, s=None):
        """The step as a list of (stage, exchange-after): stage() launches
        stream-ordered work; exchange-after names the halo segment to swap
        with the neighbour shards before the next stage (None: none).  The
        unsharded step is 8 do-alls with no exchange."""
        h, a = self.heap, self.args
        sh = self.shard is not None

        def do(T, m):
            return lambda: h.parallel_do(T, m, a, s)

        def k(kid):
            return lambda: h.launch(kid, self.W, a, s)

        def seq(*fs):
            def run():
                for f in fs:
                    f()
            return run

        def begin():
            a.step = self.step_no

        def end():
            self.step_no += 1

        out = []
        for T, dec, upd in ((FISH, dsr.M_WT_CELL_DECIDE_FISH, dsr.M_WT_FISH_UPDATE),
                            (SHARK, dsr.M_WT_CELL_DECIDE_SHARK, dsr.M_WT_SHARK_UPDATE)):
            prep = dsr.M_WT_FISH_PREPARE if T == FISH else dsr.M_WT_SHARK_PREPARE
            first = [begin] if T == FISH else []
            last = [end] if T == SHARK else []
            if not sh:
                out.append((seq(*first, do(CELL, dsr.M_WT_CELL_PREPARE), do(T, prep), do(CELL, dec), do(T, upd),
                                *last), None))
                continue
            out += [(seq(*first, do(CELL, dsr.M_WT_CELL_PREPARE), do(T, prep), k(dsr.K_WT_HALO_REQ_PACK)), "req"),
                    (seq(k(dsr.K_WT_HALO_REQ_APPLY), do(CELL, dec)), "grant"),
                    (seq(k(dsr.K_WT_HALO_GRANT_APPLY), do(T, upd)), "mig"),
                    (seq(k(dsr.K_WT_HALO_MIG_APPLY), k(dsr.K_WT_HALO_OCC_PACK)), "occ"),
                    (seq(k(dsr.K_WT_HALO_OCC_APPLY), *last), None)]
        return out

    def swap(self, seg, stream=None):
        """Exchange one halo segment with the neighbour shards (P = 1 sharded:
        with myself -- my row 1 borders my row H across the torus seam), on
        the stream the step's kernels run on."""
        with dsr.on_stream(stream if stream is not None else self.stream):
            if self.exchange is not None:
                return self.exchange(seg)
            o, i, n = self.halo_layout[seg]
            self.halo[i:i + n].copy_(self.halo[o + n:o + 2 * n])       # in[0] <- the shard above's out[1]
            self.halo[i + n:i + 2 * n].copy_(self.halo[o:o + n])       # in[1] <- the shard below's out[0]

    def step(self, stream=None):
        s = stream if stream is not None else self.stream
        for stage, seg in self.stages(s):
            stage()
            if seg is not None:
                self.swap(seg, s)

    def run(self, steps, stream=None):
        for _ in range(steps):
            self.step(stream)

    def capture(self):
        """Capture one (unsharded) step -- 8 do-alls, all stream-ordered -- as a
        CUDA graph; the step number moves to a device word that the graph
        advances itself, so replay() runs consecutive steps.  Removes the host
        launch overhead of ~24 launches per step."""
        import torch
        if self.shard is not None:
            raise ValueError("capture() is for the single-heap step (sharded steps exchange on the host)")
        dev = self.heap.device
        self.step_word = torch.tensor([self.step_no], dtype=torch.int32, device=dev)
        self.args.step_dev = self.step_word.data_ptr()
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            self.step(s)                                  # warm-up (uses and advances the device word)
            self.step_word += 1
            with torch.cuda.graph(self.graph, stream=s):
                self.step(s)
                self.step_word += 1
        torch.cuda.current_stream().wait_stream(s)
        self.step_no -= 1                                 # the captured step did not execute
        return self.graph

    def run_graph(self, steps):
        for _ in range(steps):
            self.graph.replay()
            self.step_no += 1

    def state(self, stream=None):
        """(kind, egg, energy) per cell as (H, W) numpy arrays (canonical dump)."""
        import numpy as np
        import torch
        s = stream if stream is not None else self.stream
        with torch.cuda.stream(s if s is not None else torch.cuda.current_stream()):
            self.out.zero_()
        self.heap.parallel_do(FISH, dsr.M_WT_DUMP, self.args, s)
        self.heap.parallel_do(SHARK, dsr.M_WT_DUMP, self.args, s)
        torch.cuda.synchronize()
        o = self.out.cpu().numpy().view(np.uint32).reshape(3, self.grid_rows, self.W)
        if self.shard is not None:
            o = o[:, 1:-1]                                   # local rows only
        return o[0].astype(np.uint8), o[1].copy(), o[2].copy()

    def read_counters(self):
        """Cumulative (fish born, sharks born, eaten, starved) since construction."""
        return [int(v) for v in self.counters.cpu().tolist()]


class NcclHaloExchange:
    """Wa-Tor halo segments between row-band shards over torch.distributed
    (NCCL on GPUs): out[0] (my row 1 side) goes to the shard above, out[1] to
    the shard below; in[0] / in[1] receive from above / below."""

    def __init__(self, sim, group=None):
        import torch.distributed as dist
        self.sim, self.group = sim, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def __call__(self, seg):
        import torch.distributed as dist
        if self.world == 1:
            return self._self(seg)
        o, i, n = self.sim.halo_layout[seg]
        h = self.sim.halo
        up, down = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        # posting order pairs the messages when up == down (2 ranks, no tags in NCCL)
        ops = [dist.P2POp(dist.isend, h[o + n:o + 2 * n], down, self.group),
               dist.P2POp(dist.isend, h[o:o + n], up, self.group),
               dist.P2POp(dist.irecv, h[i:i + n], up, self.group),
               dist.P2POp(dist.irecv, h[i + n:i + 2 * n], down, self.group)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()

    def _self(self, seg):
        o, i, n = self.sim.halo_layout[seg]
        h = self.sim.halo
        h[i:i + n].copy_(h[o + n:o + 2 * n])
        h[i + n:i + 2 * n].copy_(h[o:o + n])


class WaTorLoopback:
    """P row-band shards on ONE GPU (P heaps): the same stages and exchange
    points as the multi-GPU run, the messages replaced by device copies."""

    def __init__(self, kind, egg, energy, P, **kw):
        self.P = P
        self.shards = [WaTor(kind, egg, energy, shard=(r, P), **kw) for r in range(P)]

    def step(self):
        plans = [s.stages(s.stream) for s in self.shards]
        for k in range(len(plans[0])):
            for p in plans:
                p[k][0]()
            seg = plans[0][k][1]
            if seg is None:
                continue
            o, i, n = self.shards[0].halo_layout[seg]
            with dsr.StreamJoin([s.stream for s in self.shards]):
                for r, s in enumerate(self.shards):
                    up, down = self.shards[(r - 1) % self.P], self.shards[(r + 1) % self.P]
                    s.halo[i:i + n].copy_(up.halo[o + n:o + 2 * n])
                    s.halo[i + n:i + 2 * n].copy_(down.halo[o:o + n])

    def run(self, steps):
        for _ in range(steps):
            self.step()

    def state(self):
        import numpy as np
        parts = [s.state() for s in self.shards]
        return tuple(np.concatenate([p[j] for p in parts], axis=0) for j in range(3))

    def read_counters(self):
        return [sum(v) for v in zip(*(s.read_counters() for s in self.shards))]


class WaTorStatic:
    """The paper's static-allocation baseline: the same Wa-Tor rules
    on cell-indexed SOA device arrays, no heap, no objects (dsr_wator_static_step).
    Its state after any number of steps equals WaTor's bit for bit; its time
    prices the dynamic allocation."""

    def __init__(self, kind, egg, energy, FB=6, SB=12, SS=6, seed=42, device=None, stream=None, step0=0):
        import ctypes as C
        import numpy as np
        import torch
        H, W = kind.shape
        self.H, self.W, self.N = H, W, H * W
        self.device = torch.device(device if device is not None else "cuda")
        self.stream = stream
        dev = self.device
        self.kind = torch.from_numpy(np.ascontiguousarray(kind, dtype=np.uint8).ravel()).to(dev)
        self.egg = torch.from_numpy(np.ascontiguousarray(egg, dtype=np.uint32).ravel().view(np.int32)).to(dev)
        self.energy = torch.from_numpy(np.ascontiguousarray(energy, dtype=np.uint32).ravel().view(np.int32)).to(dev)
        self.target = torch.full((self.N,), -1, dtype=torch.int32, device=dev)
        self.req = torch.zeros(((self.N + 3) // 4) * 4, dtype=torch.uint8, device=dev)
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.args = dsr.WatorStaticArgs(W, H, FB, SB, SS, step0, seed, self.kind.data_ptr(), self.egg.data_ptr(),
                                        self.energy.data_ptr(), self.target.data_ptr(), self.req.data_ptr(),
                                        self.counters.data_ptr())
        self.step_no = step0
        self._C = C

    def run(self, steps, stream=None):
        s = stream if stream is not None else self.stream
        self.args.step = self.step_no
        dsr.check("dsr_wator_static_step",
                  dsr.lib().dsr_wator_static_step(self._C.byref(self.args), steps, dsr._stream_ptr(s)))
        self.step_no += steps

    def state(self):
        """(kind, egg, energy) per cell as (H, W) numpy arrays."""
        import numpy as np
        import torch
        torch.cuda.synchronize()
        k = self.kind.cpu().numpy().reshape(self.H, self.W).copy()
        e = self.egg.cpu().numpy().view(np.uint32).reshape(self.H, self.W).copy()
        n = self.energy.cpu().numpy().view(np.uint32).reshape(self.H, self.W).copy()
        return k, e, n

    def read_counters(self):
        """Cumulative (fish born, sharks born, eaten, starved)."""
        return [int(v) for v in self.counters.cpu().tolist()]
