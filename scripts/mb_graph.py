"""Microbench step: eager launches vs one CUDA graph of the whole step (same results)."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1810_11765_b200 import dsr
from paper_1810_11765_b200.microbench import Microbench

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
mb = Microbench(stream=s)
for _ in range(3):
    mb.step(stream=s)
torch.cuda.synchronize()
ref = mb.results().copy()


def timed(fn, K=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(K):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


eager = timed(lambda: mb.step(stream=s))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    mb.step(stream=s)
torch.cuda.synchronize()
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
graph = timed(g.replay)
ok = np.array_equal(mb.results(), ref) and mb.heap.poll_error() == dsr.OK and mb.heap.check_invariants() == 0
eager2 = timed(lambda: mb.step(stream=s))
print(json.dumps({"eager_ms": eager, "graph_ms": graph, "eager_again_ms": eager2, "results_equal": bool(ok)}))
