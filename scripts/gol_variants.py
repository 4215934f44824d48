"""GoL 16384^2 ms/gen per variant and pass: python scripts/gol_variants.py [gens]"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import inputs as I
from paper_1810_11765_b200.gol import GameOfLife, ALIVE, CAND

G = int(sys.argv[1]) if len(sys.argv) > 1 else 6
a0 = I.gol_soup(16384, 16384, 0.25, 42)
import os
ONLY = os.environ.get("GOL_VARIANTS", "handles,tiled_prepare,tiled_all,bits").split(",")
for name, kw in (("handles", {}), ("tiled_prepare", {"tiled": "prepare"}), ("tiled_all", {"tiled": "all"}),
                 ("bits", {"bit_mirror": True})):
    if name not in ONLY:
        continue
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    g = GameOfLife(a0, stream=s, **kw)
    g.run(1)
    torch.cuda.synchronize()
    per = []
    for _ in range(G):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        h, a = g.heap, g.args
        ev[0].record(s)
        for i, (T, m) in enumerate(((CAND, g.m[0]), (ALIVE, g.m[1]), (CAND, g.m[2]), (ALIVE, g.m[3]))):
            h.parallel_do(T, m, a, s)
            ev[i + 1].record(s)
        g.gen += 1
        torch.cuda.synchronize()
        per.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)])
    tot = [sum(p) for p in per]
    print(json.dumps({"variant": name, "ms_per_gen": tot, "passes_ms_last": per[-1],
                      "live": [g.heap.live_count(0), g.heap.live_count(1)]}), flush=True)
    del g
    torch.cuda.empty_cache()
