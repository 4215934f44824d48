import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
from paper_1810_11765_b200 import inputs as I, dsr
from paper_1810_11765_b200.gol import GameOfLife, PeerHalo
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
W, H = 96, 64
a0 = I.gol_soup(W, H, 0.3, 77)
sim = GameOfLife(a0, shard=(rank, world), peer=True)
ph = PeerHalo(sim)
F = dsr.gol_peer_flags(W)
sim.first_half(None)
torch.cuda.synchronize()
print(f"rank {rank}: after my push, my flags {sim.halo[F:F+8].cpu().numpy().view(np.uint32)}", flush=True)
dist.barrier()
time.sleep(1)
print(f"rank {rank}: after barrier, my flags {sim.halo[F:F+8].cpu().numpy().view(np.uint32)}", flush=True)
# write directly through the mapping from the host side (torch tensor from pointer is hard); use a device copy
dist.barrier()
ph.close()
dist.destroy_process_group()
