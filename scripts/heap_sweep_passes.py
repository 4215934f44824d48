"""Wa-Tor 2048^2 per-pass times (prologue / body) at two heap sizes: which
pass grows with the heap.  python scripts/heap_sweep_passes.py"""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import dsr, inputs as I
from paper_1810_11765_b200.wator import WaTor, FISH, SHARK, CELL


def timed(fn, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return round(1000 * e0.elapsed_time(e1) / reps, 1)


k, e, n = I.wator_init(2048, 2048, seed=42)
for gib in (0.5, 16):
    w = WaTor(k, e, n, heap_bytes=int(gib * (1 << 30)))
    w.run(10)
    torch.cuda.synchronize()
    h, a = w.heap, w.args
    out = {"heap_gib": gib, "M": h.M}
    seq = (("cell_prepare", CELL, dsr.M_WT_CELL_PREPARE), ("fish_prepare", FISH, dsr.M_WT_FISH_PREPARE),
           ("decide_fish", CELL, dsr.M_WT_CELL_DECIDE_FISH),
           ("shark_prepare", SHARK, dsr.M_WT_SHARK_PREPARE))
    for name, T, m in seq:      # passes that neither allocate nor destroy: repeatable
        out[name + "_prologue_us"] = timed(lambda: h.doall_prologue(T, m))
        out[name + "_us"] = timed(lambda: h.doall_body(T, m, a))
    out["step_us"] = timed(lambda: w.step(), 10)
    print(json.dumps(out), flush=True)
    del w
    torch.cuda.empty_cache()
