"""Small configurations of every app for compute-sanitizer (memcheck /
racecheck / synccheck): python scripts/sanitize_small.py.  Each result is
checked against the oracle so a run that 'passes' the tool also computed the
right thing."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from oracle import oracle as O
from paper_1810_11765_b200 import dsr, inputs as I
from paper_1810_11765_b200.microbench import Microbench
from paper_1810_11765_b200.gol import GameOfLife
from paper_1810_11765_b200.wator import WaTor
from paper_1810_11765_b200.nbody import NBody

ok = []
for bulk in (True, False):
    mb = Microbench(n1=20_000, n2=10_000, seed=3, heap_bytes=16 << 20, bulk=bulk)
    mb.step()
    torch.cuda.synchronize()
    ok.append(("microbench bulk" if bulk else "microbench per-thread",
               np.array_equal(mb.results(), O.microbench(3, 20_000, 10_000)[0]) and mb.heap.check_invariants() == 0))
a0 = I.gol_soup(64, 64, 0.3, 1)
for tiled in (False, "prepare", "all"):  # GoL
    g = GameOfLife(a0, heap_bytes=16 << 20, tiled=tiled)
    g.run(10)
    ok.append((f"gol 64 tiled={tiled}", np.array_equal(g.alive(), O.life_dense(a0, 10))))
k, e, n = I.wator_init(64, 64, seed=21)
w = WaTor(k, e, n, FB=6, SB=12, SS=6, seed=42, heap_bytes=16 << 20)
w.run(10)
gk, ge, gn = w.state()
ok.append(("wator 64", np.array_equal(gk, O.wator_run(k, e, n, FB=6, SB=12, SS=6, seed=42, steps=10)[0])))
st = I.nbody_init(1000, seed=7)
prm = dict(G=2e-9, dt=0.5, eps=0.01, R=0.02)
nb = NBody(st, merges=True, **prm)
nb.run(3)
got = nb.state()
want = O.nbody_run(st, merges=True, steps=3, **prm)
ok.append(("nbody 1000", np.array_equal(got["alive"], want["alive"])))
from paper_1810_11765_b200.gol import GameOfLifeLoopback
lbg = GameOfLifeLoopback(a0, 2, peer=True, heap_bytes=16 << 20)
lbg.run(10)
ok.append(("gol 64 two shards, peer-memory halo", np.array_equal(lbg.alive(), O.life_dense(a0, 10))))
from paper_1810_11765_b200.nbody import NBodyLoopback
st2 = I.nbody_init(1024, seed=7)
lbn = NBodyLoopback(st2, 2, merges=True, peer=True, **prm)
lbn.run(3)
one = NBody(st2, merges=True, **prm)
one.run(3)
ok.append(("nbody 1024 two shards, peer-memory all-gathers",
           all(np.array_equal(lbn.state()[k], one.state()[k]) for k in ("x", "y", "m", "alive"))))
from paper_1810_11765_b200.nbody import NBodyStatic
nbs = NBodyStatic(st, merges=True, **prm)
nbs.run(3)
ok.append(("nbody 1000 static", np.array_equal(nbs.state()["alive"], want["alive"])))
for name, v in ok:
    print(f"{name}: {'ok' if v else 'MISMATCH'}")
print("ALL OK" if all(v for _, v in ok) else "FAILED")
