"""GoL 16384^2 generation time (tiled prepare, block-list updates, as in the bench):
python scripts/ab_gol.py [gens]   (DSR_LIBPATH selects the library build)"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import inputs as I
from paper_1810_11765_b200.gol import GameOfLife

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = GameOfLife(I.gol_soup(16384, 16384, 0.25, 42), tiled="prepare")
g.run(1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.run(gens); e1.record(); torch.cuda.synchronize()
print(json.dumps({"gol16k_tiled_ms": round(e0.elapsed_time(e1) / gens, 3), "gens": gens}), flush=True)
