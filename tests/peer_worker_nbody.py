"""Worker of tests/test_gpu_apps.py::test_nbody_peer_two_processes: one N-body
id range per process, the snapshot / target all-gathers done through CUDA
IPC-mapped peer memory only (NBodyPeer); rank 0 compares the merged state with
a one-heap run (bit for bit).  Launched by torch.distributed.run (gloo)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch
import torch.distributed as dist

from paper_1810_11765_b200 import inputs as I, nbody

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)                              # both processes on one GPU (the test box has one)
st = I.nbody_init(4096, seed=11)
prm = dict(G=2e-9, dt=0.5, eps=0.01, R=0.02)
sim = nbody.NBody(st, merges=True, shard=(rank, world), peer=True, **prm)
pe = nbody.NBodyPeer(sim)
sim.run(6)
torch.cuda.synchronize()
mine = sim.state()
parts = [None] * world
dist.all_gather_object(parts, (sim.lo, sim.hi, mine))
ok = sim.heap.check_invariants() == 0
oks = [None] * world
dist.all_gather_object(oks, ok)
pe.close()
if rank == 0:
    one = nbody.NBody(st, merges=True, **prm)
    one.run(6)
    a = one.state()
    b = {k: v.copy() for k, v in parts[0][2].items()}
    for lo, hi, s in parts[1:]:
        for k in b:
            b[k][lo:hi] = s[k][lo:hi]
    assert (a["alive"] == 0).sum() > 10
    for k in ("x", "y", "vx", "vy", "m", "alive"):
        assert np.array_equal(a[k], b[k]), k
    assert all(oks)
    print("NBODY PEER OK", flush=True)
dist.barrier()
dist.destroy_process_group()
