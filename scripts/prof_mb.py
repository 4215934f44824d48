"""One instrumented microbench step: phase times and allocator counters.
usage: prof_mb.py [flags] [retries] [reserve 0/1]"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import dsr
from paper_1810_11765_b200.microbench import Microbench

flags = int(sys.argv[1]) if len(sys.argv) > 1 else dsr.F_STATS
retries = int(sys.argv[2]) if len(sys.argv) > 2 else 5
reserve = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
slack = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
mb = Microbench(flags=flags, retries=retries, reserve=reserve, reserve_slack=slack)
for _ in range(2):
    mb.step()
torch.cuda.synchronize()
mb.heap.stats_reset()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(7)]
mb.step(events=ev)
torch.cuda.synchronize()
ph = {n: round(e[0].elapsed_time(e[1]), 3) for n, e in zip(["init", "new1", "reduce2", "free3", "new4", "reduce5", "drain6"], ev)}
print(json.dumps({"flags": flags, "retries": retries, "reserve": reserve, "slack": slack, "phase_ms": ph,
                  "frag": mb.heap.fragmentation(), "stats": mb.heap.stats()}))
