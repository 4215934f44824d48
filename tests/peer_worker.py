"""Worker of tests/test_gpu_gol.py::test_gol_peer_memory_exchange_two_processes:
one GoL row-band shard per process, the halo exchanged through CUDA IPC-mapped
peer memory only (PeerHalo); rank 0 checks the assembled alive map against the
oracle's dense Life.  Launched by torch.distributed.run (gloo for the handle
exchange and the final gather)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch
import torch.distributed as dist

from paper_1810_11765_b200 import inputs as I
from paper_1810_11765_b200.gol import GameOfLife, PeerHalo

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)                              # both processes on one GPU (the test box has one)
W, H, gens = 96, 64, 40
a0 = I.gol_soup(W, H, 0.3, 77)
sim = GameOfLife(a0, shard=(rank, world), peer=True)
ph = PeerHalo(sim)
print(f"rank {rank}: mapped up/down {sim.args.peer_up:#x} {sim.args.peer_down:#x}", flush=True)
for g in range(gens):
    sim.generation()
    if os.environ.get("PEER_TRACE"):
        torch.cuda.synchronize()
        print(f"rank {rank}: generation {g} done", flush=True)
torch.cuda.synchronize()
mine = sim.alive()
parts = [None] * world
dist.all_gather_object(parts, mine)
ok = sim.heap.check_invariants() == 0
oks = [None] * world
dist.all_gather_object(oks, ok)
ph.close()
if rank == 0:
    from oracle import oracle as O
    O.build()
    got = np.concatenate(parts, axis=0)
    want = O.life_dense(a0, gens)
    assert np.array_equal(got, want), "peer-memory exchange differs from dense Life"
    assert all(oks)
    print("PEER OK", flush=True)
dist.barrier()
dist.destroy_process_group()
