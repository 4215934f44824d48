"""N-body with collisions driver (Table 1, Listing 1; reading
R-NBODY).  One step = snapshot S0, compute_force (device_do as a tiled
all-pairs gather), move, snapshot S1, prepare_merge, claim, absorb,
delete_merged.  BASELINE configs[2] (65,536 fp32 bodies).

Multi-GPU (one process per GPU, `group` = a torch.distributed process group):
rank r owns ids [r n/P, (r+1) n/P) in its own heap; after each snapshot the
S/V chunks are all-gathered, after prepare_merge the target chunk; the claim
then runs redundantly over all ids on every rank (O(n)), so absorption and
deletion need no third exchange and the result does not depend on P.
"""
from __future__ import annotations

from . import dsr

NB_TYPES = [[4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 1]]   # x y vx vy fx fy m id target incoming merged
NONE = 0xFFFFFFFF


def id_range(n_total: int, world: int, rank: int):
    """Ids owned by `rank` (contiguous equal chunks; n_total % world == 0)."""
    if n_total % world:
        raise ValueError("n_total must be divisible by the number of ranks")
    c = n_total // world
    return rank * c, (rank + 1) * c


class Exchange:
    """All-gathers of the id-indexed arrays between the ranks' heaps."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0

    def all_gather_rows(self, full, lo, hi):
        """full: tensor whose first dim is id; rows [lo, hi) are this rank's."""
        if self.world == 1:
            return
        import torch.distributed as dist
        chunk = full[lo:hi].contiguous()
        dist.all_gather_into_tensor(full, chunk, group=self.group)


class NBody:
    def __init__(self, state, G, dt, eps, R, merges=True, heap_bytes=None, device=None, stream=None, group=None,
                 n_total=None, shard=None, peer=False):
        """state: dict of x, y, vx, vy, m for ALL ids (each rank keeps its chunk).
        shard = (rank, world) emulates a rank without a process group (loopback).
        peer: the all-gathers are the snapshot pass's own stores into every
        peer's (epoch-parity) buffers plus flags (dsr.h "Peer-memory
        all-gathers"); connect() sets the peers' buffers first."""
        import numpy as np
        import torch
        self.xch = Exchange(group)
        self.rank, self.world = shard if shard is not None else (self.xch.rank, self.xch.world)
        N = n_total or len(state["x"])
        self.n_total = N
        self.lo, self.hi = id_range(N, self.world, self.rank)
        n = self.hi - self.lo
        self.merges = merges
        if heap_bytes is None:
            heap_bytes = max(8 << 20, n * 64 + (8 << 20))
        self.heap = dsr.Heap(NB_TYPES, heap_bytes, device=device, stream=stream)
        dev = self.heap.device
        self.stream = stream
        f = lambda k: torch.from_numpy(np.ascontiguousarray(state[k][self.lo:self.hi], np.float32)).to(dev)
        self.init = {k: f(k) for k in ("x", "y", "vx", "vy", "m")}
        self.S = torch.zeros(N, 4, dtype=torch.float32, device=dev)
        self.V = torch.zeros(N, 2, dtype=torch.float32, device=dev)
        self.target = torch.full((N,), -1, dtype=torch.int32, device=dev)
        self.incoming = torch.full((N,), -1, dtype=torch.int32, device=dev)
        self.shandle = torch.zeros(N, dtype=torch.int64, device=dev)
        self.out = torch.zeros(N, 6, dtype=torch.float32, device=dev)
        chunks = (N + 4095) // 4096
        self.scratch = torch.zeros(2 * chunks * n, dtype=torch.float32, device=dev)
        self.live = torch.zeros(4 * N + chunks, dtype=torch.float32, device=dev)   # all-pairs live list (dsr.h)
        i = self.init
        self.args = dsr.NbodyArgs(self.S.data_ptr(), self.V.data_ptr(), self.target.data_ptr(),
                                  self.incoming.data_ptr(), self.shandle.data_ptr(),
                                  i["x"].data_ptr(), i["y"].data_ptr(), i["vx"].data_ptr(), i["vy"].data_ptr(),
                                  i["m"].data_ptr(), G, dt, eps, R, N, self.lo, self.hi, self.out.data_ptr(),
                                  self.scratch.data_ptr(), self.live.data_ptr())
        self.heap.parallel_new(0, n, dsr.C_NB_BODY, self.args, stream)
        self.peer = bool(peer) and self.world > 1
        self.epoch = 0                              # snapshots taken (2 per step)
        self.step_no = 0
        if self.peer:
            # double buffers by epoch (S, V) and step (target) parity; flags: 2 x world u32
            self.S2 = [self.S, torch.zeros_like(self.S)]
            self.V2 = [self.V, torch.zeros_like(self.V)]
            self.T2 = [self.target, torch.full_like(self.target, -1)]
            self.flags = torch.zeros(2 * self.world, dtype=torch.int32, device=dev)
            a = self.args
            a.npeers, a.rank, a.world, a.flags = self.world - 1, self.rank, self.world, self.flags.data_ptr()
            self.peers = None

    def peer_buffers(self):
        """This rank's exchanged buffers (for the peers to map): S[2], V[2], target[2], flags."""
        return {"S": self.S2, "V": self.V2, "target": self.T2, "flags": self.flags}

    def connect(self, peers):
        """peers[i]: device pointers {"S": [p0, p1], "V": [...], "target": [...], "flags": p} of rank
        (rank + 1 + i) % world (other shards' buffers on this GPU, or IPC-mapped ones)."""
        assert self.peer and len(peers) == self.world - 1
        self.peers = peers

    def _peer_args(self, e=None, k=None):
        a = self.args
        if e is not None:
            a.S, a.V, a.epoch = self.S2[e & 1].data_ptr(), self.V2[e & 1].data_ptr(), e
            for i, p in enumerate(self.peers):
                a.peer_S[i], a.peer_V[i], a.peer_flags[i] = p["S"][e & 1], p["V"][e & 1], p["flags"]
        if k is not None:
            a.target = self.T2[k & 1].data_ptr()
            for i, p in enumerate(self.peers):
                a.peer_target[i] = p["target"][k & 1]

    # ---- one step as a sequence of local phases ("p") and exchange points ("x")
    def sequence(self):
        seq = ["p_snapshot", "x_SV", "p_force_move"]                       # S0, compute_force, move
        if self.merges:
            seq += ["p_snapshot", "x_SV", "p_merge_search", "x_target", "p_claim_absorb_delete"]
        return seq

    def p_snapshot(self, s):
        h, a = self.heap, self.args
        if self.peer:
            if self.epoch % 2 == 0:                 # a step begins: its target buffer
                self._peer_args(k=self.step_no)
            self._peer_args(e=self.epoch)
        h.launch(dsr.K_NB_CLEAR_SNAPSHOT, self.n_total, a, s)
        h.parallel_do(0, dsr.M_NB_SNAPSHOT, a, s)
        if self.peer:
            h.launch(dsr.K_NB_SIGNAL, self.n_total, a, s)
            self.epoch += 1

    def p_force_move(self, s):
        self.heap.parallel_do(0, dsr.M_NB_FORCE, self.args, s)
        self.heap.parallel_do(0, dsr.M_NB_MOVE, self.args, s)

    def p_merge_search(self, s):
        self.heap.parallel_do(0, dsr.M_NB_PREPARE_MERGE, self.args, s)

    def p_claim_absorb_delete(self, s):
        h, a = self.heap, self.args
        if self.peer:
            a.epoch = self.step_no                   # the claim waits for the peers' target rows of this step
        if self.world > 1:
            h.launch(dsr.K_NB_CLAIM, self.n_total, a, s)       # over the gathered targets of all ids
        else:
            h.parallel_do(0, dsr.M_NB_CLAIM, a, s)
        h.parallel_do(0, dsr.M_NB_ABSORB, a, s)
        h.parallel_do(0, dsr.M_NB_DELETE_MERGED, a, s)
        if self.peer:
            self.args.epoch = self.epoch - 1         # (only the target exchange used the step number)
        self.step_no += 1

    def _push_target(self, s):
        a = self.args
        a.epoch = self.step_no
        self.heap.launch(dsr.K_NB_PUSH_TARGET, self.n_total, a, s)

    def x_SV(self, s=None):
        if self.peer:
            return                                   # the snapshot pass wrote every peer's rows
        with dsr.on_stream(s if s is not None else self.stream):   # in order with the kernels on s
            self.xch.all_gather_rows(self.S, self.lo, self.hi)
            self.xch.all_gather_rows(self.V, self.lo, self.hi)

    def x_target(self, s=None):
        if self.peer:
            self._push_target(s if s is not None else self.stream)   # my rows into every peer's target + flags
            return
        with dsr.on_stream(s if s is not None else self.stream):
            self.xch.all_gather_rows(self.target, self.lo, self.hi)

    def step(self, stream=None):
        s = stream if stream is not None else self.stream
        for name in self.sequence():
            getattr(self, name)(s)

    def run(self, steps, stream=None):
        for _ in range(steps):
            self.step(stream)

    def state(self, stream=None):
        """id-indexed dict x, y, vx, vy, m (float32) and alive (uint8) of this rank's ids
        (all ids on one GPU)."""
        import numpy as np
        import torch
        s = stream if stream is not None else self.stream
        with torch.cuda.stream(s if s is not None else torch.cuda.current_stream()):
            self.out.zero_()
        self.heap.parallel_do(0, dsr.M_NB_DUMP, self.args, s)
        torch.cuda.synchronize()
        o = self.out.cpu().numpy()
        return {"x": o[:, 0].copy(), "y": o[:, 1].copy(), "vx": o[:, 2].copy(), "vy": o[:, 3].copy(),
                "m": o[:, 4].copy(), "alive": (o[:, 5] > 0).astype(np.uint8)}


class NBodyStatic:
    """The paper's static-allocation baseline of N-body: the same
    passes on id-indexed SOA arrays, no heap (dsr_nbody_static_step); its
    state after any number of steps equals NBody's bit for bit."""

    def __init__(self, state, G, dt, eps, R, merges=True, device=None, stream=None):
        import ctypes as C
        import numpy as np
        import torch
        n = len(state["x"])
        dev = torch.device(device if device is not None else "cuda")
        self.n, self.stream, self._C = n, stream, C
        S = np.zeros((n, 4), np.float32)
        alive = np.asarray(state.get("alive", np.ones(n, np.uint8))) != 0
        S[:, 0], S[:, 1], S[:, 2] = state["x"], state["y"], np.where(alive, state["m"], 0)
        self.S = torch.from_numpy(S).to(dev)
        self.V = torch.from_numpy(np.stack([state["vx"], state["vy"]], 1).astype(np.float32)).to(dev)
        self.target = torch.full((n,), -1, dtype=torch.int32, device=dev)
        self.incoming = torch.full((n,), -1, dtype=torch.int32, device=dev)
        self.scratch = torch.zeros(2 * ((n + 4095) // 4096) * n, dtype=torch.float32, device=dev)
        self.live = torch.zeros(4 * n + (n + 4095) // 4096, dtype=torch.float32, device=dev)
        self.args = dsr.NbodyStaticArgs(self.S.data_ptr(), self.V.data_ptr(), self.target.data_ptr(),
                                        self.incoming.data_ptr(), self.scratch.data_ptr(), G, dt, eps, R, n,
                                        1 if merges else 0, self.live.data_ptr())

    def run(self, steps, stream=None):
        s = stream if stream is not None else self.stream
        dsr.check("dsr_nbody_static_step", dsr.lib().dsr_nbody_static_step(self._C.byref(self.args), steps,
                                                                           dsr._stream_ptr(s)))

    def state(self):
        import numpy as np
        import torch
        torch.cuda.synchronize()
        S, V = self.S.cpu().numpy(), self.V.cpu().numpy()
        alive = (S[:, 2] > 0).astype(np.uint8)
        z = lambda v: np.where(alive == 1, v, 0).astype(np.float32)
        return {"x": z(S[:, 0]), "y": z(S[:, 1]), "vx": z(V[:, 0]), "vy": z(V[:, 1]), "m": z(S[:, 2]), "alive": alive}


class NBodyPeer:
    """Multi-process peer mode: every rank exports its exchanged buffers (S and
    V of both epoch parities, target of both step parities, flags) as CUDA IPC
    handles, all-gathers them over torch.distributed and maps every other
    rank's (over NVLink / NVSwitch when they are other GPUs)."""

    def __init__(self, sim, group=None):
        import torch.distributed as dist
        assert sim.peer, "NBody(..., peer=True) under a process group of > 1 ranks"
        bufs = sim.peer_buffers()
        mine = {k: ([dsr.ipc_handle(t) for t in v] if isinstance(v, list) else dsr.ipc_handle(v))
                for k, v in bufs.items()}
        allh = [None] * sim.world
        dist.all_gather_object(allh, mine, group=group)
        self.opened = []
        bases = {}                                  # one mapping per exported block (a caching allocator
                                                    # may put several buffers in one block)

        def open_(hd):
            h, off = hd
            if h not in bases:
                bases[h] = dsr.ipc_open(h)
                self.opened.append(bases[h])
            return bases[h] + off
        peers = []
        for i in range(sim.world - 1):
            r = (sim.rank + 1 + i) % sim.world
            peers.append({k: ([open_(x) for x in v] if isinstance(v, list) else open_(v)) for k, v in allh[r].items()})
        sim.connect(peers)
        dist.barrier(group)

    def close(self):
        for p in self.opened:
            dsr.ipc_close(p)
        self.opened = []


class NBodyLoopback:
    """P id-range shards of the N-body step on ONE GPU: P heaps, the same
    kernels and phase order as the multi-GPU run, the all-gathers replaced by
    device-to-device copies of each shard's rows into every other shard's
    id-indexed arrays.  Used to test the sharded algorithm without P GPUs."""

    def __init__(self, state, P, **kw):
        self.shards = [NBody(state, shard=(r, P), **kw) for r in range(P)]
        if self.shards[0].peer:                      # peer mode: each shard writes into the others' buffers
            bufs = [sh.peer_buffers() for sh in self.shards]
            ptrs = [{"S": [t.data_ptr() for t in b["S"]], "V": [t.data_ptr() for t in b["V"]],
                     "target": [t.data_ptr() for t in b["target"]], "flags": b["flags"].data_ptr()} for b in bufs]
            for r, sh in enumerate(self.shards):
                sh.connect([ptrs[(r + 1 + i) % P] for i in range(P - 1)])

    def _gather(self, attr):
        src = self.shards
        for dst in src:
            for s in src:
                if s is not dst:
                    getattr(dst, attr)[s.lo:s.hi].copy_(getattr(s, attr)[s.lo:s.hi])

    def step(self):
        for name in self.shards[0].sequence():
            if name.startswith("p_"):
                for sh in self.shards:
                    getattr(sh, name)(sh.stream)
            elif self.shards[0].peer:
                if name == "x_target":              # push every shard's rows before any claim waits for them
                    for sh in self.shards:
                        sh.x_target(sh.stream)
            elif name == "x_SV":
                self._gather("S")
                self._gather("V")
            else:
                self._gather("target")

    def run(self, steps):
        for _ in range(steps):
            self.step()

    def state(self):
        """Merge the shards' dumps (each shard dumps only its own ids)."""
        import numpy as np
        out = None
        for sh in self.shards:
            st = sh.state()
            if out is None:
                out = {k: v.copy() for k, v in st.items()}
            else:
                sel = np.zeros(len(out["x"]), bool)
                sel[sh.lo:sh.hi] = True
                for k in out:
                    out[k][sel] = st[k][sel]
        return out
