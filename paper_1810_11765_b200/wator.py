"""Wa-Tor driver: the host loop of eight dsr_parallel_do calls per step
(Table 1; reading R-WATOR).  BASELINE configs[1] (2048^2, 500 steps)."""
from __future__ import annotations

from . import dsr

WT_TYPES = [[4, 4, 4], [4, 4, 4, 4], [4, 8, 1, 1, 1, 1, 1]]   # Fish, Shark, Cell
FISH, SHARK, CELL = 0, 1, 2


class WaTor:
    def __init__(self, kind, egg, energy, FB=6, SB=12, SS=6, seed=42, heap_bytes=None, device=None,
                 stream=None, retries=5, flags=0, step0=0):
        import numpy as np
        import torch
        H, W = kind.shape
        self.W, self.H, self.N = W, H, W * H
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
        self.args = dsr.WatorArgs(self.cells.data_ptr(), W, H, FB, SB, SS, seed, step0,
                                  self.kind0.data_ptr(), self.egg0.data_ptr(), self.energy0.data_ptr(),
                                  self.out[0].data_ptr(), self.out[1].data_ptr(), self.out[2].data_ptr(),
                                  self.counters.data_ptr())
        self.heap.parallel_new(CELL, self.N, dsr.C_WT_CELL, self.args, stream)   # constructor i -> id i
        self.heap.launch(dsr.K_WT_INIT_AGENTS, self.N, self.args, stream)
        self.step_no = step0

    def step(self, stream=None):
        s = stream if stream is not None else self.stream
        h, a = self.heap, self.args
        a.step = self.step_no
        h.parallel_do(CELL, dsr.M_WT_CELL_PREPARE, a, s)
        h.parallel_do(FISH, dsr.M_WT_FISH_PREPARE, a, s)
        h.parallel_do(CELL, dsr.M_WT_CELL_DECIDE_FISH, a, s)
        h.parallel_do(FISH, dsr.M_WT_FISH_UPDATE, a, s)
        h.parallel_do(CELL, dsr.M_WT_CELL_PREPARE, a, s)
        h.parallel_do(SHARK, dsr.M_WT_SHARK_PREPARE, a, s)
        h.parallel_do(CELL, dsr.M_WT_CELL_DECIDE_SHARK, a, s)
        h.parallel_do(SHARK, dsr.M_WT_SHARK_UPDATE, a, s)
        self.step_no += 1

    def run(self, steps, stream=None):
        for _ in range(steps):
            self.step(stream)

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
        o = self.out.cpu().numpy().view(np.uint32)
        return (o[0].astype(np.uint8).reshape(self.H, self.W), o[1].reshape(self.H, self.W),
                o[2].reshape(self.H, self.W))

    def read_counters(self):
        """Cumulative (fish born, sharks born, eaten, starved) since construction."""
        return [int(v) for v in self.counters.cpu().tolist()]
