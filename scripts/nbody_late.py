"""N-body 65536 per-phase times after s steps (clustering changes the merge search's
slow-path rate): python scripts/nbody_late.py"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import dsr, inputs as I
from paper_1810_11765_b200.nbody import NBody


def timed(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


sim = NBody(I.nbody_init(65536, 7), merges=True, **I.NBODY_PARAMS)
done = 0
for upto in (2, 100, 300, 600, 900):
    sim.run(upto - done)
    done = upto
    h, a = sim.heap, sim.args
    out = {"step": done, "bodies": h.live_count(0)}
    sim.p_snapshot(None)
    out["force"] = timed(lambda: h.parallel_do(0, dsr.M_NB_FORCE, a))
    out["merge_search"] = timed(lambda: h.parallel_do(0, dsr.M_NB_PREPARE_MERGE, a))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sim.run(5); e1.record(); torch.cuda.synchronize()
    done += 5
    out["step_ms"] = round(e0.elapsed_time(e1) / 5, 4)
    print(json.dumps(out), flush=True)
