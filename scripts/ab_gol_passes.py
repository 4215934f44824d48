"""GoL 16384^2 (tiled prepare) per-pass device times over generations 2-4:
python scripts/ab_gol_passes.py   (DSR_LIBPATH selects the library build)"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import inputs as I
from paper_1810_11765_b200.gol import GameOfLife, ALIVE, CAND

g = GameOfLife(I.gol_soup(16384, 16384, 0.25, 42), tiled="prepare")
g.run(1)
torch.cuda.synchronize()
types = (CAND, ALIVE, CAND, ALIVE)
ms = [0.0] * 4
for gen in range(3):
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.heap.parallel_do(types[i], g.m[i], g.args)
        e1.record()
        torch.cuda.synchronize()
        ms[i] += e0.elapsed_time(e1) / 3
print(json.dumps({"pass_ms": [round(x, 3) for x in ms], "gen_ms": round(sum(ms), 3)}), flush=True)
