"""Wa-Tor 2048^2 agent fragmentation F and populations every 25 steps
of the 500-step run: python scripts/wator_frag_trace.py [r]  (DSR_LIBPATH selects the build)"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import inputs as I
from paper_1810_11765_b200.wator import WaTor, FISH, SHARK
from scripts.ablation import agent_frag

r = int(sys.argv[1]) if len(sys.argv) > 1 else 5
kind, egg, en = I.wator_init(2048, 2048, seed=42)
sim = WaTor(kind, egg, en, seed=42, retries=r)
trace = []
for step in range(0, 500, 25):
    sim.run(25)
    torch.cuda.synchronize()
    f, b = agent_frag(sim.heap, [FISH, SHARK])
    trace.append([step + 25, round(f, 4), sim.heap.live_count(FISH), sim.heap.live_count(SHARK), b])
print(json.dumps({"r": r, "sms": None, "trace": trace}), flush=True)
