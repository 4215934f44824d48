"""N-body with collisions driver (Table 1, Listing 1; reading
R-NBODY).  One step = snapshot S0, compute_force (device_do as a tiled
all-pairs gather), move, snapshot S1, prepare_merge, claim, absorb,
delete_merged.  BASELINE configs[2] (65,536 fp32 bodies)."""
from __future__ import annotations

from . import dsr

NB_TYPES = [[4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 1]]   # x y vx vy fx fy m id target incoming merged


class NBody:
    def __init__(self, state, G, dt, eps, R, merges=True, heap_bytes=None, device=None, stream=None, id_offset=0,
                 n_total=None):
        import numpy as np
        import torch
        n = len(state["x"])
        self.n = n
        self.n_total = n_total or n
        self.merges = merges
        if heap_bytes is None:
            heap_bytes = max(8 << 20, n * 64 + (8 << 20))
        self.heap = dsr.Heap(NB_TYPES, heap_bytes, device=device, stream=stream)
        dev = self.heap.device
        self.stream = stream
        f = lambda k: torch.from_numpy(np.ascontiguousarray(state[k], np.float32)).to(dev)
        self.init = {k: f(k) for k in ("x", "y", "vx", "vy", "m")}
        N = self.n_total
        self.S = torch.zeros(5, N, dtype=torch.float32, device=dev)     # x y m vx vy
        self.shandle = torch.zeros(N, dtype=torch.int64, device=dev)
        self.out = torch.zeros(N, 6, dtype=torch.float32, device=dev)
        S = self.S
        self.args = dsr.NbodyArgs(S[0].data_ptr(), S[1].data_ptr(), S[2].data_ptr(), S[3].data_ptr(),
                                  S[4].data_ptr(), self.shandle.data_ptr(),
                                  self.init["x"].data_ptr(), self.init["y"].data_ptr(), self.init["vx"].data_ptr(),
                                  self.init["vy"].data_ptr(), self.init["m"].data_ptr(), G, dt, eps, R, N,
                                  id_offset, self.out.data_ptr())
        self.heap.parallel_new(0, n, dsr.C_NB_BODY, self.args, stream)

    def snapshot(self, s=None):
        h, a = self.heap, self.args
        h.launch(dsr.K_NB_CLEAR_SNAPSHOT, self.n_total, a, s)
        h.parallel_do(0, dsr.M_NB_SNAPSHOT, a, s)

    def step(self, stream=None):
        s = stream if stream is not None else self.stream
        h, a = self.heap, self.args
        self.snapshot(s)                                   # S0
        h.parallel_do(0, dsr.M_NB_FORCE, a, s)
        h.parallel_do(0, dsr.M_NB_MOVE, a, s)
        if not self.merges:
            return
        self.snapshot(s)                                   # S1
        h.parallel_do(0, dsr.M_NB_PREPARE_MERGE, a, s)
        h.parallel_do(0, dsr.M_NB_CLAIM, a, s)
        h.parallel_do(0, dsr.M_NB_ABSORB, a, s)
        h.parallel_do(0, dsr.M_NB_DELETE_MERGED, a, s)

    def run(self, steps, stream=None):
        for _ in range(steps):
            self.step(stream)

    def state(self, stream=None):
        """id-indexed dict x, y, vx, vy, m (float32) and alive (uint8)."""
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
