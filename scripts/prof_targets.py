"""Minimal drivers for ncu captures: python scripts/prof_targets.py mb|nbody|gol16k[-tiled|-tiledall|-bits]|wator
The library build (src hash) is written to gpurun_out/build_info.txt for the summaries."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import inputs as I

w = sys.argv[1]
if w == "none":
    pass
elif w == "mb":
    from paper_1810_11765_b200.microbench import Microbench
    mb = Microbench()
    for _ in range(2):
        mb.step()
elif w == "nbody":
    from paper_1810_11765_b200.nbody import NBody
    sim = NBody(I.nbody_init(65536, 7), merges=True, **I.NBODY_PARAMS)
    sim.run(3)
elif w.startswith("gol16k"):
    from paper_1810_11765_b200.gol import GameOfLife
    kw = {"gol16k-tiled": {"tiled": "prepare"}, "gol16k-tiledall": {"tiled": "all"},
          "gol16k-bits": {"bit_mirror": True}}.get(w, {})
    g = GameOfLife(I.gol_soup(16384, 16384, 0.25, 42), **kw)
    g.run(3)
elif w == "wator":
    from paper_1810_11765_b200.wator import WaTor
    k, e, n = I.wator_init(2048, 2048, seed=42)
    sim = WaTor(k, e, n)
    sim.run(4)
torch.cuda.synchronize()
import os
from paper_1810_11765_b200 import dsr
os.makedirs('gpurun_out', exist_ok=True)
open('gpurun_out/build_info.txt', 'w').write(dsr.lib().dsr_build_info().decode())
