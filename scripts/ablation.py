"""Ablations and sweeps on B200 (the paper's §6 design
claims): NoShift / NoCoal / NoCoal-NoShift, the active-block lookup
attempts r, heap size and the Linux Scalability n-sweep
(P:918-923), on the allocator microbenchmark (configs[4]) and Wa-Tor 2048^2
(configs[1], the paper's ablation app).

usage: python scripts/ablation.py [out.jsonl]      (driver: one subprocess per
       configuration, each under a timeout, so a pathological ablation cannot
       hang the run)
       python scripts/ablation.py --one KIND JSON  (one configuration)"""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

FLAGS = {"default": 0, "NoShift": 0x1, "NoCoal": 0x2, "NoCoal-NoShift": 0x3, "NoHint": 0x10, "SlotRotate": 0x80,
         "QuadFree": 0x200, "BulkDense": 0x400}


def agent_frag(heap, types):
    """F = 1 - live / (blocks x N_T) over the given types."""
    _, blocks = heap.fragmentation()
    slots = sum(blocks[t] * heap.cap[t] for t in types)
    live = sum(heap.live_count(t) for t in types)
    return (1.0 - live / slots) if slots else 0.0, [blocks[t] for t in types]


def one_mb(cfg):
    import torch
    from paper_1810_11765_b200 import dsr
    from paper_1810_11765_b200.microbench import Microbench
    n1, n2 = cfg.get("n1", 1 << 26), cfg.get("n2", 1 << 25)
    mb = Microbench(n1=n1, n2=n2, flags=cfg["flags"], retries=cfg["r"], reserve=cfg["reserve"],
                    heap_bytes=cfg.get("heap_bytes"), bulk=cfg.get("bulk", False))
    mb.step()                                          # warm-up
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(7)]
        mb.step(events=ev)
        torch.cuda.synchronize()
        times.append([e[0].elapsed_time(e[1]) for e in ev])
    med = [sorted(t[i] for t in times)[1] for i in range(7)]
    # fragmentation after phase 4 (untimed replay of phases 1, 3, 4)
    h = mb.heap
    h.reset()
    if cfg["reserve"]:
        for t, c in enumerate(mb._counts(0, n1)):
            h.reserve_blocks(t, -(-c // h.cap[t]))
    h.launch(mb.kernel, n1, dsr.MbNewArgs(1, 0))
    if cfg["reserve"]:
        for t in range(3):
            h.trim(t)
    f1, b1 = agent_frag(h, [0, 1, 2])
    for t in range(3):
        h.parallel_do(t, dsr.M_MB_FREE_ODD, None)
    h.launch(mb.kernel, n2, dsr.MbNewArgs(1, n1))
    f4, b4 = agent_frag(h, [0, 1, 2])
    assert h.poll_error() == dsr.OK
    names = ["init", "new1", "reduce2", "free3", "new4", "reduce5", "drain6"]
    return {"phase_ms": dict(zip(names, [round(x, 3) for x in med])), "step_ms": round(sum(med), 3),
            "allocs_per_s_new1": n1 / (med[1] * 1e-3), "frag_after_new1": f1, "frag_after_new4": f4,
            "blocks_after_new4": b4}


def one_wator(cfg):
    import torch
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.wator import WaTor, FISH, SHARK
    W = cfg.get("W", 2048)
    kind, egg, en = I.wator_init(W, W, seed=42)
    sim = WaTor(kind, egg, en, seed=42, flags=cfg["flags"], retries=cfg["r"], heap_bytes=cfg.get("heap_bytes"))
    steps = cfg.get("steps", 500)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.run(steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    f, b = agent_frag(sim.heap, [FISH, SHARK])
    from paper_1810_11765_b200 import dsr
    err = sim.heap.poll_error()
    return {"ms_per_step": round(ms, 4), "steps": steps, "agent_frag": f, "agent_blocks": b,
            "device_error": dsr.status_str(err),
            "fish": sim.heap.live_count(FISH), "sharks": sim.heap.live_count(SHARK)}


def one_ls(cfg):
    import numpy as np
    import torch
    from paper_1810_11765_b200 import dsr
    n, threads = cfg["n"], 16384
    heap = dsr.Heap([[4] * 16], 1 << 30, flags=cfg.get("flags", 0))
    handles = torch.zeros(threads * n, dtype=torch.int64, device="cuda")
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record()
    heap.launch(dsr.K_LS_ALLOC, threads, dsr.LsArgs(handles.data_ptr(), n, 0))
    e[1].record()
    heap.launch(dsr.K_LS_FREE, threads, dsr.LsArgs(handles.data_ptr(), n, 0))
    e[2].record()
    torch.cuda.synchronize()
    h = handles.cpu().numpy()
    ok = int((h != 0).sum())
    err = heap.poll_error()
    cap_objs = (1 << 30) // 64
    return {"alloc_ms": round(e[0].elapsed_time(e[1]), 4), "free_ms": round(e[1].elapsed_time(e[2]), 4),
            "alloc_us_per_obj_per_thread": e[0].elapsed_time(e[1]) * 1e3 / n,
            "allocated": ok, "requested": threads * n, "oom": err == dsr.ERR_OOM,
            "utilisation_of_heap": ok * 64 / (1 << 30), "objects_fit_if_perfect": cap_objs}


def runs():
    if os.environ.get("ABL_ONLY") == "wator-noshift":
        return [("wator", {"name": n, "flags": FLAGS[n], "r": 5, **hb}) for n in ("NoShift", "NoCoal-NoShift")
                for hb in ({}, {"heap_bytes": 4 << 30})]
    out = []
    # the bench's allocation kernel (warp-cooperative, R-BULK) and its free-pass ablation (R-BLOCKDOALL)
    out.append(("mb", {"name": "bulk (bench default)", "flags": 0, "r": 5, "reserve": False, "bulk": True}))
    out.append(("mb", {"name": "bulk, QuadFree", "flags": FLAGS["QuadFree"], "r": 5, "reserve": False, "bulk": True}))
    out.append(("mb", {"name": "bulk, NoShift", "flags": FLAGS["NoShift"], "r": 5, "reserve": False, "bulk": True}))
    out.append(("mb", {"name": "bulk, BulkDense", "flags": FLAGS["BulkDense"], "r": 5, "reserve": False, "bulk": True}))
    # the paper-shaped per-thread kernel (one Alg. 1 request per coalesced lane group) under the paper's ablations
    for name in ["default", "NoShift", "NoCoal", "NoCoal-NoShift", "NoHint", "SlotRotate"]:
        out.append(("mb", {"name": name, "flags": FLAGS[name], "r": 5, "reserve": True}))
    out.append(("mb", {"name": "paper-exact (NoHint, SlotRotate, no reserve)", "flags": 0x90, "r": 5, "reserve": False}))
    out.append(("mb", {"name": "default, no reserve", "flags": 0, "r": 5, "reserve": False}))
    for r in [1, 2, 3, 8]:
        out.append(("mb", {"name": f"r={r}", "flags": 0, "r": r, "reserve": True}))
    for name in ["default", "NoShift", "NoCoal", "NoCoal-NoShift", "NoHint", "SlotRotate"]:
        out.append(("wator", {"name": name, "flags": FLAGS[name], "r": 5}))
    for r in [1, 2, 3, 8]:
        out.append(("wator", {"name": f"r={r}", "flags": 0, "r": r}))
    for gb in [0.5, 1, 2, 4, 8, 16]:
        out.append(("wator", {"name": f"heap {gb} GiB", "flags": 0, "r": 5, "heap_bytes": int(gb * (1 << 30)),
                              "steps": 200}))
    for n in [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]:
        out.append(("ls", {"name": f"linux-scalability n={n}", "n": n}))
    return out


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        kind, cfg = sys.argv[2], json.loads(sys.argv[3])
        res = {"mb": one_mb, "wator": one_wator, "ls": one_ls}[kind](cfg)
        print("RESULT " + json.dumps(res), flush=True)
        return
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ablation.jsonl"
    with open(path, "w") as f:
        for kind, cfg in runs():
            t = time.time()
            try:
                p = subprocess.run([sys.executable, __file__, "--one", kind, json.dumps(cfg)], capture_output=True,
                                   text=True, timeout=150)
                lines = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
                res = json.loads(lines[-1][7:]) if lines else {"error": (p.stderr or "")[-400:]}
            except subprocess.TimeoutExpired:
                res = {"error": "timeout 150 s"}
            rec = {"workload": kind, **cfg, **res, "wall_s": round(time.time() - t, 1)}
            f.write(json.dumps(rec) + "\n")
            f.flush()
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
