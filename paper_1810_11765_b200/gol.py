"""Game of Life (O(#alive) Alive/Candidate version) driver: the host loop of
four dsr_parallel_do calls per generation (Table 1; reading R-GOL).
BASELINE configs[0] (64x64, 100 generations) and configs[3] (16384^2)."""
from __future__ import annotations

from . import dsr

GOL_TYPES = [[4, 1, 1], [4, 1]]      # Alive{cell, is_new, action}, Candidate{cell, action}
ALIVE, CAND = 0, 1


class GameOfLife:
    def __init__(self, alive0, heap_bytes=None, device=None, stream=None, retries=5, flags=0):
        import numpy as np
        import torch
        H, W = alive0.shape
        self.W, self.H, self.N = W, H, W * H
        if heap_bytes is None:
            # every cell could hold an object: 5-6 B per object in 53/64-slot blocks, x2 slack
            heap_bytes = max(16 << 20, self.N * 2 * 384 // 53 + (8 << 20))
        self.heap = dsr.Heap(GOL_TYPES, heap_bytes, device=device, retries=retries, flags=flags, stream=stream)
        dev = self.heap.device
        self.stream = stream
        self.cell = torch.zeros(self.N, dtype=torch.int64, device=dev)
        self.alive0 = torch.from_numpy(np.ascontiguousarray(alive0, dtype=np.uint8).reshape(-1)).to(dev)
        self.dumpbuf = torch.zeros(self.N, dtype=torch.int32, device=dev)
        self.args = dsr.GolArgs(self.cell.data_ptr(), W, H, self.alive0.data_ptr(), self.dumpbuf.data_ptr())
        self.heap.launch(dsr.K_GOL_INIT_ALIVE, self.N, self.args, stream)
        self.heap.launch(dsr.K_GOL_INIT_CAND, self.N, self.args, stream)
        self.gen = 0

    def generation(self, stream=None):
        s = stream if stream is not None else self.stream
        h, a = self.heap, self.args
        h.parallel_do(CAND, dsr.M_GOL_CAND_PREPARE, a, s)
        h.parallel_do(ALIVE, dsr.M_GOL_ALIVE_PREPARE, a, s)
        h.parallel_do(CAND, dsr.M_GOL_CAND_UPDATE, a, s)
        h.parallel_do(ALIVE, dsr.M_GOL_ALIVE_UPDATE, a, s)
        self.gen += 1

    def run(self, gens, stream=None):
        for _ in range(gens):
            self.generation(stream)

    def capture(self):
        """Capture one generation (4 do-alls = memsets + compaction + method
        kernels, all stream-ordered, no host synchronisation) as a CUDA graph;
        replay it with run_graph().  Small grids are launch-bound, so this
        removes ~14 launches of host overhead per generation."""
        import torch
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
        return self.dumpbuf.cpu().numpy().reshape(self.H, self.W)

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
