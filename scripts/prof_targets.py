"""Minimal drivers for ncu captures: python scripts/prof_targets.py mb|nbody|gol16k|wator"""
import sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import inputs as I

w = sys.argv[1]
if w == "mb":
    from paper_1810_11765_b200.microbench import Microbench
    mb = Microbench()
    for _ in range(2):
        mb.step()
elif w == "nbody":
    from paper_1810_11765_b200.nbody import NBody
    sim = NBody(I.nbody_init(65536, 7), merges=True, **I.NBODY_PARAMS)
    sim.run(3)
elif w == "gol16k":
    from paper_1810_11765_b200.gol import GameOfLife
    g = GameOfLife(I.gol_soup(16384, 16384, 0.25, 42))
    g.run(2)
elif w == "wator":
    from paper_1810_11765_b200.wator import WaTor
    k, e, n = I.wator_init(2048, 2048, seed=42)
    sim = WaTor(k, e, n)
    sim.run(4)
torch.cuda.synchronize()
