"""Per-pass CUDA-event timings of the app workloads (diagnostics)."""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_1810_11765_b200 import dsr, inputs as I

def timed(fn, reps=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)

which = sys.argv[1:] or ["gol16k", "wator", "nbody"]
if "gol16k" in which:
    from paper_1810_11765_b200.gol import GameOfLife, ALIVE, CAND
    g = GameOfLife(I.gol_soup(16384, 16384, 0.25, 42))
    h, a = g.heap, g.args
    for gen in range(3):
        out = {"gen": gen, "alive": h.live_count(ALIVE), "cand": h.live_count(CAND)}
        for name, T, m in (("cand_prepare", CAND, dsr.M_GOL_CAND_PREPARE), ("alive_prepare", ALIVE, dsr.M_GOL_ALIVE_PREPARE),
                           ("cand_update", CAND, dsr.M_GOL_CAND_UPDATE), ("alive_update", ALIVE, dsr.M_GOL_ALIVE_UPDATE)):
            out[name + "_prologue"] = timed(lambda: h.doall_prologue(T, m))
            out[name] = timed(lambda: h.doall_body(T, m, a))
        print(json.dumps(out), flush=True)
if "wator" in which:
    from paper_1810_11765_b200.wator import WaTor, FISH, SHARK, CELL
    k, e, n = I.wator_init(2048, 2048, seed=42)
    w = WaTor(k, e, n)
    w.run(5)
    h, a = w.heap, w.args
    out = {"fish": h.live_count(FISH), "sharks": h.live_count(SHARK)}
    seq = (("cell_prepare", CELL, dsr.M_WT_CELL_PREPARE), ("fish_prepare", FISH, dsr.M_WT_FISH_PREPARE),
           ("decide_fish", CELL, dsr.M_WT_CELL_DECIDE_FISH), ("fish_update", FISH, dsr.M_WT_FISH_UPDATE),
           ("cell_prepare2", CELL, dsr.M_WT_CELL_PREPARE), ("shark_prepare", SHARK, dsr.M_WT_SHARK_PREPARE),
           ("decide_shark", CELL, dsr.M_WT_CELL_DECIDE_SHARK), ("shark_update", SHARK, dsr.M_WT_SHARK_UPDATE))
    a.step = w.step_no
    for name, T, m in seq:
        out[name + "_prologue"] = timed(lambda: h.doall_prologue(T, m))
        out[name] = timed(lambda: h.doall_body(T, m, a))
    print(json.dumps(out), flush=True)
if "nbody" in which:
    from paper_1810_11765_b200.nbody import NBody
    sim = NBody(I.nbody_init(65536, 7), merges=True, **I.NBODY_PARAMS)
    sim.run(2)
    h, a = sim.heap, sim.args
    out = {}
    out["clear"] = timed(lambda: h.launch(dsr.K_NB_CLEAR_SNAPSHOT, sim.n_total, a))
    out["snapshot"] = timed(lambda: h.parallel_do(0, dsr.M_NB_SNAPSHOT, a))
    out["force"] = timed(lambda: h.parallel_do(0, dsr.M_NB_FORCE, a), 3)
    out["merge_search"] = timed(lambda: h.parallel_do(0, dsr.M_NB_PREPARE_MERGE, a), 3)
    out["step"] = timed(sim.step, 3)
    out["pairs_per_s_force"] = 65536 ** 2 / (out["force"] * 1e-3)
    print(json.dumps(out), flush=True)
