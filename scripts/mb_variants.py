"""Microbench step times of the allocation variants (bulk / per-thread / +reserve).
python scripts/mb_variants.py [reps]"""
import json, sys, statistics
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import dsr
from paper_1810_11765_b200.microbench import Microbench, PHASES

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["bulk", "scalar_doall", "per_thread", "per_thread_reserve"]
V = {"bulk": dict(bulk=True), "scalar_doall": dict(bulk=True, flags=dsr.F_SCALAR_DOALL),
     "quad_free": dict(bulk=True, flags=dsr.F_QUAD_FREE),
     "per_thread": dict(bulk=False), "per_thread_reserve": dict(bulk=False, reserve=True)}
for name in which:
    kw = V[name]
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    mb = Microbench(stream=s, **kw)
    for _ in range(2):
        mb.step()
    torch.cuda.synchronize()
    ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(7)] for _ in range(reps)]
    for k in range(reps):
        mb.step(events=ev[k])
    torch.cuda.synchronize()
    ph = {p: round(statistics.median(ev[k][i][0].elapsed_time(ev[k][i][1]) for k in range(reps)), 4)
          for i, p in enumerate(PHASES)}
    assert mb.heap.poll_error() == dsr.OK
    print(json.dumps({"variant": name, "lib": str(dsr.LIBPATH.name), "step_ms": round(sum(ph.values()), 4), "phases": ph,
                      "frag_blocks": mb.heap.fragmentation()[1]}), flush=True)
    del mb
    torch.cuda.empty_cache()
