"""A/B of allocator flags on the app workloads: python scripts/ab_apps.py FLAGS [wator|gol16k ...]"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import inputs as I

flags = int(sys.argv[1])
which = sys.argv[2:] or ["wator", "gol16k"]


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


out = {"flags": flags}
if "wator" in which:
    from paper_1810_11765_b200.wator import WaTor
    k, e, n = I.wator_init(2048, 2048, seed=42)
    w = WaTor(k, e, n, flags=flags)
    w.run(20)
    out["wator_ms"] = timed(lambda: w.run(1), 50)
    out["wator_frag"] = w.heap.fragmentation()[0]
if "gol16k" in which:
    from paper_1810_11765_b200.gol import GameOfLife
    g = GameOfLife(I.gol_soup(16384, 16384, 0.25, 42), flags=flags)
    g.run(1)
    out["gol16k_ms"] = timed(lambda: g.run(1), 3)
print(json.dumps(out), flush=True)
