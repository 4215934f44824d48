"""Wa-Tor 2048^2 ms/step vs heap size (do-all enumeration cost should
not depend on the heap size).  python scripts/heap_sweep.py"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import inputs as I
from paper_1810_11765_b200.wator import WaTor

k, e, n = I.wator_init(2048, 2048, seed=42)
import os
for gib in [float(x) for x in os.environ.get("HEAP_GIB", "0.5,2,8,16").split(",")]:
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    w = WaTor(k, e, n, heap_bytes=int(gib * (1 << 30)), stream=s)
    w.run(10)
    w.capture()
    for _ in range(5):
        w.graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(50):
        w.graph.replay()
    e1.record(s)
    torch.cuda.synchronize()
    print(json.dumps({"heap_gib": gib, "M": w.heap.M, "ms_per_step": e0.elapsed_time(e1) / 50,
                      "frag": w.heap.fragmentation()[0]}), flush=True)
    del w
    torch.cuda.empty_cache()
