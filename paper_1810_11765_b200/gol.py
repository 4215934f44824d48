"""Game of Life (O(#alive) Alive/Candidate version) driver: the host loop of
four dsr_parallel_do calls per generation (Table 1; reading R-GOL).
BASELINE configs[0] (64x64, 100 generations) and configs[3] (16384^2)."""
from __future__ import annotations

from . import dsr

GOL_TYPES = [[4, 1, 1], [4, 1]]      # Alive{cell, is_new, action}, Candidate{cell, action}
ALIVE, CAND = 0, 1


def row_range(H: int, world: int, rank: int):
    """Rows owned by `rank` (contiguous bands; H % world == 0)."""
    if H % world:
        raise ValueError("H must be divisible by the number of shards")
    b = H // world
    return rank * b, (rank + 1) * b


class GameOfLife:
    """One heap for the whole torus, or -- with shard=(rank, P) -- one row band
    of it with two ghost rows: after pass 3 the boundary rows'
    next-alive / new-alive masks go to the neighbouring shards (`exchange`),
    which store them as ghost rows and create the Candidates on their own
    boundary cells next to a remote new Alive.  With P shards the result is the
    single-heap result bit for bit."""

    def __init__(self, alive0, heap_bytes=None, device=None, stream=None, retries=5, flags=0, shard=None,
                 exchange=None, bit_mirror=False, tiled=False, peer=False):
        """tiled: True / "prepare" -- the two prepare passes (the neighbour
        gathers) as cell-tiled do-alls (DSR_M_GOL_*_PREPARE_TILED: objects
        enumerated through the cell grid, neighbour handles staged in shared
        memory), the update passes on the block list (full warps, destroys and
        news coalesced per block); "all" -- all four passes cell-tiled.  Same
        results as the block-list passes."""
        import numpy as np
        import torch
        Hg, W = alive0.shape
        self.Hg = Hg
        self.shard = shard
        if shard is not None:
            r, P = shard
            y0, y1 = row_range(Hg, P, r)
            self.y0, self.y1 = y0, y1
            H = y1 - y0
            rows = [(y0 - 1) % Hg] + list(range(y0, y1)) + [y1 % Hg]
            grid = np.ascontiguousarray(alive0[rows], dtype=np.uint8)
            self.grid_rows = H + 2
        else:
            self.y0, self.y1, H = 0, Hg, Hg
            grid = np.ascontiguousarray(alive0, dtype=np.uint8)
            self.grid_rows = H
        self.W, self.H, self.N = W, H, W * self.grid_rows
        self.exchange = exchange
        if heap_bytes is None:
            # every cell could hold an object: 5-6 B per object in 53/64-slot blocks, x2 slack
            heap_bytes = max(16 << 20, W * H * 2 * 384 // 53 + (8 << 20))
        self.heap = dsr.Heap(GOL_TYPES, heap_bytes, device=device, retries=retries, flags=flags, stream=stream)
        dev = self.heap.device
        self.stream = stream
        self.cell = torch.zeros(self.N, dtype=torch.int64, device=dev)
        self.alive0 = torch.from_numpy(grid.reshape(-1)).to(dev)
        self.dumpbuf = torch.zeros(self.N, dtype=torch.int32, device=dev)
        self.halo = torch.zeros(4 * W, dtype=torch.uint8, device=dev)
        # variant: alive-bit mirror read by the prepare passes (1 bit per cell instead of 8-B handles)
        self.bits = torch.zeros(self.grid_rows * ((W + 31) // 32), dtype=torch.int32, device=dev) if bit_mirror \
            else None
        self.args = dsr.GolArgs(self.cell.data_ptr(), W, H, self.alive0.data_ptr(), self.dumpbuf.data_ptr(),
                                1 if shard is not None else 0, self.halo.data_ptr() if shard is not None else None,
                                self.bits.data_ptr() if bit_mirror else None)
        # peer: the halo is exchanged through peer memory (DSR_K_GOL_HALO_PUSH writes my boundary masks
        # straight into the neighbours' halo buffers, dsr.h "Peer-memory halo exchange"); connect() sets
        # the neighbours' buffers before the first generation
        self.peer = bool(peer) and shard is not None
        if self.peer:
            self.halo = torch.zeros(dsr.gol_peer_halo_bytes(W), dtype=torch.uint8, device=dev)
            self.args.halo = self.halo.data_ptr()
        if tiled and bit_mirror:
            raise ValueError("tiled passes read the handle grid; the bit mirror is the other variant")
        if tiled == "all":
            self.m = (dsr.M_GOL_CAND_PREPARE_TILED, dsr.M_GOL_ALIVE_PREPARE_TILED, dsr.M_GOL_CAND_UPDATE_TILED,
                      dsr.M_GOL_ALIVE_UPDATE_TILED)
        elif tiled:
            self.m = (dsr.M_GOL_CAND_PREPARE_TILED, dsr.M_GOL_ALIVE_PREPARE_TILED, dsr.M_GOL_CAND_UPDATE,
                      dsr.M_GOL_ALIVE_UPDATE)
        else:
            self.m = (dsr.M_GOL_CAND_PREPARE, dsr.M_GOL_ALIVE_PREPARE, dsr.M_GOL_CAND_UPDATE, dsr.M_GOL_ALIVE_UPDATE)
        self.heap.launch(dsr.K_GOL_INIT_ALIVE, self.N, self.args, stream)
        self.heap.launch(dsr.K_GOL_INIT_CAND, self.N, self.args, stream)
        self.gen = 0

    def connect(self, peer_up: int, peer_down: int):
        """Peer mode: device pointers of the halo buffers of the shards above
        and below (another shard's `halo` on this GPU, or an IPC-mapped one)."""
        self.args.peer_up, self.args.peer_down = peer_up, peer_down

    # the generation split at the exchange point (sharded mode)
    def first_half(self, s):
        h, a = self.heap, self.args
        h.parallel_do(CAND, self.m[0], a, s)
        h.parallel_do(ALIVE, self.m[1], a, s)
        h.parallel_do(CAND, self.m[2], a, s)
        if self.peer:
            a.gen = self.gen
            h.launch(dsr.K_GOL_HALO_PUSH, self.W, a, s)
        elif self.shard is not None:
            h.launch(dsr.K_GOL_HALO_PACK, self.W, a, s)

    def second_half(self, s):
        h, a = self.heap, self.args
        if self.shard is not None:
            h.launch(dsr.K_GOL_HALO_APPLY, self.W, a, s)
        h.parallel_do(ALIVE, self.m[3], a, s)
        self.gen += 1

    def generation(self, stream=None):
        s = stream if stream is not None else self.stream
        self.first_half(s)
        if self.shard is not None and not self.peer:
            with dsr.on_stream(s):                  # the copies / NCCL calls in order with the kernels on s
                (self.exchange or self.self_exchange)()
        self.second_half(s)

    def self_exchange(self):
        """P = 1 sharded mode: my bottom row is my top ghost row and vice versa."""
        W = self.W
        self.halo[2 * W:3 * W].copy_(self.halo[W:2 * W])
        self.halo[3 * W:4 * W].copy_(self.halo[0:W])

    def run(self, gens, stream=None):
        for _ in range(gens):
            self.generation(stream)

    def capture(self):
        """Capture one generation (4 do-alls = memsets + compaction + method
        kernels, all stream-ordered, no host synchronisation) as a CUDA graph;
        replay it with run_graph().  Small grids are launch-bound, so this
        removes ~14 launches of host overhead per generation."""
        import torch
        if self.peer:
            raise ValueError("peer-mode generations carry their generation number in the launch arguments "
                             "(the flags' target); they are not graph-replayable")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            self.generation(s)                      # warm-up outside the capture
            with torch.cuda.graph(self.graph, stream=s):
                self.generation(s)
        torch.cuda.current_stream().wait_stream(s)
        self.gen -= 1                               # the captured generation did not execute
        return self.graph

    def run_graph(self, gens):
        for _ in range(gens):
            self.graph.replay()
            self.gen += 1

    def dump(self, stream=None):
        """Per-cell canonical state: int32 kind | is_new << 8 | action << 16 (0 = empty)."""
        import torch
        s = stream if stream is not None else self.stream
        with torch.cuda.stream(s if s is not None else torch.cuda.current_stream()):
            self.dumpbuf.zero_()
        self.heap.parallel_do(ALIVE, dsr.M_GOL_DUMP, self.args, s)
        self.heap.parallel_do(CAND, dsr.M_GOL_DUMP, self.args, s)
        torch.cuda.synchronize()
        d = self.dumpbuf.cpu().numpy().reshape(self.grid_rows, self.W)
        return d[1:-1] if self.shard is not None else d       # local rows only

    def alive(self, stream=None):
        return ((self.dump(stream) & 0xFF) == 1).astype("uint8")

    def records(self, stream=None):
        """Canonical records sorted by cell: (cell, kind, is_new, action) -- the
        oracle's dump format."""
        import numpy as np
        d = self.dump(stream).reshape(-1)
        c = np.nonzero(d)[0]
        v = d[c]
        return np.stack([c, v & 0xFF, (v >> 8) & 0xFF, (v >> 16) & 0xFF], axis=1).astype(np.uint32)


class GameOfLifeStatic:
    """The paper's static-allocation baseline of Game of Life: B3/S23
    on a u8 cell grid, no objects (dsr_gol_static_step)."""

    def __init__(self, alive0, device=None, stream=None):
        import ctypes as C
        import numpy as np
        import torch
        self.H, self.W = alive0.shape
        dev = torch.device(device if device is not None else "cuda")
        self.cur = torch.from_numpy(np.ascontiguousarray(alive0, dtype=np.uint8).reshape(-1)).to(dev)
        self.next = torch.zeros_like(self.cur)
        self.stream, self._C = stream, C
        self.args = dsr.GolStaticArgs(self.W, self.H, self.cur.data_ptr(), self.next.data_ptr())

    def run(self, gens, stream=None):
        s = stream if stream is not None else self.stream
        dsr.check("dsr_gol_static_step", dsr.lib().dsr_gol_static_step(self._C.byref(self.args), gens,
                                                                       dsr._stream_ptr(s)))

    def alive(self):
        import torch
        torch.cuda.synchronize()
        return self.cur.cpu().numpy().reshape(self.H, self.W)


class NcclHaloExchange:
    """Halo exchange between row-band shards over torch.distributed (NCCL on
    GPUs): my first row's masks go to the shard above, my last row's to the
    shard below (torus of ranks)."""

    def __init__(self, sim, group=None):
        import torch.distributed as dist
        self.sim, self.group = sim, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def __call__(self):
        import torch.distributed as dist
        W, h = self.sim.W, self.sim.halo
        if self.world == 1:
            return self.sim.self_exchange()
        up, down = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        # messages between one pair are matched in posting order (no tags in
        # NCCL): with two ranks up == down, so the order below pairs "my last
        # row -> the lower shard's top ghost" before "my first row -> the upper
        # shard's bottom ghost" on both sides
        ops = [dist.P2POp(dist.isend, h[W:2 * W], down, self.group),
               dist.P2POp(dist.isend, h[0:W], up, self.group),
               dist.P2POp(dist.irecv, h[2 * W:3 * W], up, self.group),
               dist.P2POp(dist.irecv, h[3 * W:4 * W], down, self.group)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()


class PeerHalo:
    """Multi-process peer mode: every rank exports its halo buffer as a CUDA IPC
    handle, the handles are all-gathered over torch.distributed (any backend),
    and each rank maps its two neighbours' buffers (over NVLink / NVSwitch when
    they are on other GPUs) into its kernel arguments.  After that no host
    exchange happens: DSR_K_GOL_HALO_PUSH writes into the neighbours' memory and
    DSR_K_GOL_HALO_APPLY waits on the flags they set."""

    def __init__(self, sim, group=None):
        import torch.distributed as dist
        assert sim.peer, "GameOfLife(..., peer=True)"
        self.sim = sim
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        handles = [None] * world
        dist.all_gather_object(handles, dsr.ipc_handle(sim.halo), group=group)
        up, down = (rank - 1) % world, (rank + 1) % world
        self.opened = []

        def ptr(r):
            if r == rank:
                return sim.halo.data_ptr()
            hd, off = handles[r]
            p = dsr.ipc_open(hd)
            self.opened.append(p)
            return p + off
        mapped = {r: ptr(r) for r in {up, down}}
        sim.connect(mapped[up], mapped[down])
        dist.barrier(group)                         # every rank mapped its neighbours before the first push

    def close(self):
        for p in self.opened:
            dsr.ipc_close(p)
        self.opened = []


class GameOfLifeLoopback:
    """P row-band shards on ONE GPU (P heaps): the same kernels and exchange
    points as the multi-GPU run, the messages replaced by device copies."""

    def __init__(self, alive0, P, **kw):
        self.P = P
        self.shards = [GameOfLife(alive0, shard=(r, P), **kw) for r in range(P)]
        if self.shards[0].peer:                     # peer mode: each shard pushes into its neighbours' halos
            for r, s in enumerate(self.shards):
                s.connect(self.shards[(r - 1) % P].halo.data_ptr(), self.shards[(r + 1) % P].halo.data_ptr())

    def generation(self):
        for s in self.shards:
            s.first_half(s.stream)
        if self.shards[0].peer:
            # the pushes of every shard precede every apply in stream order (one
            # stream per shard would need the events below; the apply kernels wait
            # on the flags anyway)
            with dsr.StreamJoin([s.stream for s in self.shards]):
                pass
            for s in self.shards:
                s.second_half(s.stream)
            return
        W = self.shards[0].W
        with dsr.StreamJoin([s.stream for s in self.shards]):
            for r, s in enumerate(self.shards):
                up, down = self.shards[(r - 1) % self.P], self.shards[(r + 1) % self.P]
                s.halo[2 * W:3 * W].copy_(up.halo[W:2 * W])       # the upper shard's last row
                s.halo[3 * W:4 * W].copy_(down.halo[0:W])         # the lower shard's first row
        for s in self.shards:
            s.second_half(s.stream)

    def run(self, gens):
        for _ in range(gens):
            self.generation()

    def alive(self):
        import numpy as np
        return np.concatenate([s.alive() for s in self.shards], axis=0)
