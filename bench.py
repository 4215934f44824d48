#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the DynaSOAr B200 hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload microbench]

Workload (BASELINE.json configs[4], SURVEY c.4 / §8(d) D5): the allocator
microbenchmark -- one step = heap init, device new of 2^26 objects over three
types (12/16/24 B), do-all field reduction of every type, do-all self-delete of
the odd half, device new of 2^25 more, reduction again, do-all drain.  This is
one pass over every §8(a) row of the allocation + do-all hot path on one
batch; see DESIGN.md "Bench workload" for why it (and not the L2-resident
Wa-Tor config) is the N=1 bench line.  Multi-GPU: one heap per GPU, identical
work per rank, no data-path collective ("weak" scaling).

value = object-updates/s of the whole job: every object touched by the step
(each device new, each destroy, each do-all visit counts once) / max-over-ranks
device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "object-updates/s per app + do-all HBM GB/s vs 8 TB/s peak; allocs/s"
N1, N2, SEED = 1 << 26, 1 << 25, 1
CONFIG = {"workload": "microbench (BASELINE configs[4]): per GPU 2^26 + 2^25 device new over "
                      "A{3xu32}/B{4xu32}/C{6xu32}, 2 do-all reductions, do-all odd-free, do-all drain",
          "n1": N1, "n2": N2, "seed": SEED,
          "l2": "inputs larger than L2 (1.5 GiB live SOA data per step vs 126 MB L2); heap re-initialised every step"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="microbench", choices=["microbench", "wator", "gol", "gol16k", "gol16k-bits", "nbody"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes (read + write) of the roofline kernels from the
    committed `ncu --set full` summary (profiles/<round>/ncu_summary.json)."""
    out = {}
    for p in sorted((ROOT / "profiles").glob("r*/ncu_summary.json")):
        try:
            rows = json.loads(p.read_text())
        except Exception:
            continue
        for key in ("k_mb_new", "k_mb_reduce"):
            v = [r["dram_bytes"] for r in rows if key in r.get("kernel", "") and "dram_bytes" in r]
            if v:
                out[key] = sum(v) / len(v)
            v = [r["inst_executed"] for r in rows if key in r.get("kernel", "") and "inst_executed" in r]
            if v:
                out[key + ":inst"] = sum(v) / len(v)
            v = [r["l2_atom_alu_requests"] for r in rows if key in r.get("kernel", "") and "l2_atom_alu_requests" in r]
            if v:
                out[key + ":atom"] = sum(v) / len(v)
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init(n):
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def reduce_over_ranks(vals, op, device="cuda"):
    """Sum ("sum") or max ("max") of a list of floats over all ranks (identity
    without an initialised process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(vals)
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)
    return t.tolist()


# ---------------------------------------------------------------- CPU oracle leg
def oracle_sample(steps=1, warmup=0, n1=N1, n2=N2):
    """The oracle (oracle/, plain C, one thread) on the microbench workload
    (n1 / n2 = a bounded sample of it); returns object-updates per step and the
    per-step wall times."""
    from oracle import oracle as O
    O.build()
    for _ in range(warmup):
        O.microbench(SEED, n1, n2)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        out, live = O.microbench(SEED, n1, n2)
        ts.append(time.perf_counter() - t0)
    ph2, ph5 = int(out[0, :, 0].sum()), int(out[1, :, 0].sum())
    updates = (n1 + n2) + (ph2 + n2 - ph5 + ph5) + 2 * ph2 + 2 * ph5
    return updates, ts


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    # each step: a quarter of the workload (2^24 + 2^23, same phases), so the
    # default --steps/--warmup run stays within a few minutes on one core
    updates, ts = oracle_sample(args.steps, args.warmup, N1 // 4, N2 // 4)
    t = sum(ts) / len(ts)
    v = updates / t
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "object-updates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": CONFIG,
        "cpu_baseline": {"value": v, "unit": "object-updates/s", "cores": 1, "kind": "oracle",
                         "sample": f"each step: the microbench phases on n1 = 2^24, n2 = 2^23 (a quarter of the "
                                   f"workload), oracle/ plain C single-threaded object store, {t:.2f} s/step"},
        "e2e": {"value": v, "unit": "object-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU leg
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1810_11765_b200 import build, dsr
    from paper_1810_11765_b200.microbench import MB_TYPES, Microbench

    rank, world, local = dist_init(args.gpus)
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA GPU (no CPU fallback)")
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    mb = Microbench(n1=N1, n2=N2, seed=SEED, stream=stream)
    sizes = [sum(f) for f in MB_TYPES]
    caps = mb.heap.cap

    def step(ev=None, body_ev=None):
        mb.step(stream=stream, events=ev, body_events=body_ev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert mb.heap.poll_error() == dsr.OK, "device error during warm-up"

    # L2 atomic peak (roofline denominator of the allocator's atomics): the
    # library's probe, hashed independent u64 atomicOr-with-return over a
    # 32 MiB (L2-resident) buffer, timed with events; best of 3
    abuf = torch.zeros(4 << 20, dtype=torch.int64, device="cuda")
    dsr.probe_atomics(abuf, 0, 64, stream)
    atom_rates = []
    for _ in range(3):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        nops = dsr.probe_atomics(abuf, 0, 256, stream)
        a1.record(stream)
        torch.cuda.synchronize()
        atom_rates.append(nops / (a0.elapsed_time(a1) * 1e-3))
    atom_peak = max(atom_rates)
    del abuf

    K = args.steps
    phase_ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(7)] for _ in range(K)]
    body_ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(6)] for _ in range(K)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else local)
    launches0 = dsr.kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0.record(stream)
    for k in range(K):
        step(phase_ev[k], body_ev[k])
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = dsr.kernel_launches() - launches0
    ms = t0.elapsed_time(t1) / K
    assert mb.heap.poll_error() == dsr.OK, "device error in timed region"

    # correctness of the timed work (closed-form check happens in tests; here: drain + counts)
    res = mb.results()
    counts = mb.counts()
    updates = counts["allocs"] + counts["frees"] + counts["visits"]
    phase_ms = [statistics.mean(phase_ev[k][i][0].elapsed_time(phase_ev[k][i][1]) for k in range(K)) for i in range(7)]
    body_ms = [statistics.mean(body_ev[k][i][0].elapsed_time(body_ev[k][i][1]) for k in range(K)) for i in range(6)]

    # blocks per type at the two reductions (one extra, untimed, instrumented step)
    blocks = []
    mb.heap.reset(stream)
    mb.out.zero_()
    mb.heap.launch(mb.kernel, N1, dsr.MbNewArgs(SEED, 0), stream)
    blocks.append(mb.heap.fragmentation(stream)[1])
    for t in range(3):
        mb.heap.parallel_do(t, dsr.M_MB_FREE_ODD, None, stream)
    mb.heap.launch(mb.kernel, N2, dsr.MbNewArgs(SEED, N1), stream)
    frag5, b5 = mb.heap.fragmentation(stream)
    blocks.append(b5)
    # algorithmic bytes of the reduce bodies: live x size_T + 12 B per block
    body_bytes = []
    for ph, blk in ((0, blocks[0]), (1, blocks[1])):
        for t in range(3):
            body_bytes.append(int(res[ph, t, 0]) * sizes[t] + 12 * int(blk[t]))
    scan_bytes = sum(body_bytes)
    scan_ms = sum(body_ms)
    scan_gbs = scan_bytes / (scan_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    # dominant kernel: k_mb_new (device new + constructor).  Algorithmic bytes =
    # the constructed objects' fields + 16 B per block initialised (type id +
    # object bitmap); its two launches are exactly phases new1 / new4.
    per_type = lambda n: [(n + 1) // 2, n // 4 + (1 if n % 4 > 2 else 0), n // 4]   # [A,A,B,C][t&3]
    new_bytes = sum(c * s for c, s in zip(per_type(N1), sizes)) + sum(c * s for c, s in zip(per_type(N2), sizes))
    new_bytes += 16 * (sum(int(b) for b in blocks[1]))
    new_ms = phase_ms[1] + phase_ms[4]
    new_gbs = new_bytes / (new_ms * 1e-3) / 1e9
    traffic = ncu_traffic()

    # ---- e2e through the C ABI with HOST buffers: every step passes the host
    # (pinned) arrays of its 2^26 + 2^25 new objects' field values
    # (inputs.mb_fields, 1.61 GB) to dsr_launch(K_MB_NEW, in_host = 1), which
    # copies them into the heap's device staging buffers on its own copy stream
    # (overlapping the work already queued), and reads the 144-byte result back.
    from paper_1810_11765_b200 import inputs as I
    in1_h = torch.from_numpy(I.mb_fields(SEED, 0, N1).view(np.int32)).pin_memory()
    in2_h = torch.from_numpy(I.mb_fields(SEED, N1, N2).view(np.int32)).pin_memory()
    hres = torch.empty(18, dtype=torch.int64).pin_memory()
    h2d_bytes = in1_h.numel() * 4 + in2_h.numel() * 4

    def e2e_steps(n):
        for _ in range(n):
            mb.step(stream=stream, inputs=(in1_h.data_ptr(), in2_h.data_ptr()), host_inputs=True)
            hres.copy_(mb.out, non_blocking=True)

    e2e_steps(1)
    torch.cuda.synchronize()
    e2e_res = hres.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    e2e_steps(K)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / K
    assert np.array_equal(e2e_res.numpy().view(np.uint64).reshape(2, 3, 3), res), \
        "host-input step differs from the device-key step"

    # ---- aggregate over ranks (max time, sum of work)
    tot_updates, = reduce_over_ranks([float(updates)], "sum")
    ms_max, e2e_max = reduce_over_ranks([ms, e2e_ms], "max")
    value = tot_updates / (ms_max * 1e-3)
    e2e_value = tot_updates / (e2e_max * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            up_c, ts = oracle_sample(1, 0)
            cpu = {"value": up_c / ts[0], "unit": "object-updates/s", "cores": 1, "kind": "oracle",
                   "sample": f"full workload once (n1=2^26, n2=2^25), {ts[0]:.1f} s single-threaded"}
        except Exception as e:   # the bench line must still print
            cpu = {"value": None, "unit": "object-updates/s", "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "object-updates/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": dict(CONFIG, heap_bytes=mb.heap.buf.numel(), M=mb.heap.M, caps=caps,
                           parallelism=f"{world} independent heaps (one per GPU)"),
            "allocs_per_s": (N1 + N2) * world / (sum(phase_ms[i] for i in (1, 4)) * 1e-3),
            "frees_per_s": counts["frees"] * world / (sum(phase_ms[i] for i in (3, 6)) * 1e-3),
            "scan_gbs": scan_gbs,
            "phase_ms": dict(zip(["init", "new1", "reduce2", "free3", "new4", "reduce5", "drain6"], phase_ms)),
            "fragmentation_after_phase4": frag5,
            "roofline": {"bound": "hbm", "kernel": "k_mb_new (device new + constructors, 2 launches/step; "
                                                     f"{100 * new_ms / ms:.0f}% of the step)",
                         "achieved": new_gbs, "peak": peak, "unit": "GB/s", "frac": new_gbs / peak,
                         "traffic": traffic.get("k_mb_new"), "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": new_bytes / 2,
                         "note": "latency/contention-bound on the shared active-block bitmaps, not HBM"},
            # the allocation kernel is instruction-issue bound (ncu: issue slots ~80 % busy): warp
            # instructions per new1 launch (committed ncu --set full summary) / live new1 time, against
            # 148 SMs x 4 schedulers x 1 warp-instruction/clk at the sampled SM clock
            "roofline_issue": None if "k_mb_new:inst" not in traffic or not clk.get("sm_mhz") else {
                "bound": "issue", "kernel": "k_mb_new (phase new1 launch)",
                "achieved": traffic["k_mb_new:inst"] / (phase_ms[1] * 1e-3) / 1e9,
                "peak": 148 * 4 * clk["sm_mhz"] * 1e6 / 1e9, "unit": "G warp-inst/s",
                "frac": traffic["k_mb_new:inst"] / (phase_ms[1] * 1e-3) / (148 * 4 * clk["sm_mhz"] * 1e6),
                "inst_per_launch": traffic["k_mb_new:inst"],
                "note": "instruction count from the committed ncu summary of the same build (profiles/)"},
            # the allocation kernel's L2 atomics (ncu request count of the same build, per new1
            # launch) against the measured L2 atomic peak: not the bound, reported per SURVEY §8(d)
            "roofline_atomics": {
                "bound": "l2_atomics", "kernel": "k_mb_new (phase new1 launch)",
                "achieved": traffic["k_mb_new:atom"] / (phase_ms[1] * 1e-3) / 1e9 if "k_mb_new:atom" in traffic else None,
                "peak": atom_peak / 1e9, "unit": "G atomics/s",
                "frac": traffic["k_mb_new:atom"] / (phase_ms[1] * 1e-3) / atom_peak if "k_mb_new:atom" in traffic else None,
                "atomics_per_alloc": traffic["k_mb_new:atom"] / N1 if "k_mb_new:atom" in traffic else None,
                "peak_source": "measured in this run: dsr_probe_atomics, hashed u64 atomicOr with return over 32 MiB"},
            "roofline_scan": {"bound": "hbm", "kernel": "k_mb_reduce<NF> (do-all field scan body, 6 launches/step; "
                                                        "the BASELINE >= 60% target)",
                              "achieved": scan_gbs, "peak": peak, "unit": "GB/s", "frac": scan_gbs / peak,
                              "traffic": traffic.get("k_mb_reduce"), "peak_source": peak_src,
                              "algorithmic_bytes_per_launch": scan_bytes / 6},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "object-updates/s", "h2d_bytes_per_step": h2d_bytes,
                    "d2h_bytes_per_step": 144,
                    "what": "dsr_launch with HOST buffers: the new objects' field values (pinned host memory) "
                            "staged H2D by the library every step on its copy stream, result read back"},
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- per-app lines (not the default)
def time_steps(step, K, W, stream, per_step=None):
    """W untimed steps, then K steps between CUDA events on `stream`; returns ms/step."""
    import torch
    for _ in range(W):
        step()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(K):
        step()
        if per_step is not None:
            per_step(k)
    t1.record(stream)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / K


def run_app(args):
    """Object-updates/s of one BASELINE app config at N = 1 (diagnostic lines;
    the driver's bench line is the microbenchmark)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1810_11765_b200 import dsr, inputs as I
    rank, world, local = dist_init(args.gpus)
    if world > 1 and args.workload not in ("nbody", "gol16k", "gol16k-bits", "wator"):
        raise SystemExit(f"--workload {args.workload} runs on one GPU (replicas only); use nbody, gol16k, wator "
                         "or microbench")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    K, W = args.steps, args.warmup
    live = torch.zeros(K, 3, dtype=torch.int64, device="cuda")
    if args.workload == "wator":
        from paper_1810_11765_b200.wator import WaTor, NcclHaloExchange as WtExchange
        kind, egg, en = I.wator_init(2048, 2048, seed=42)
        if world > 1:                      # row bands + NCCL P2P boundary exchanges
            sim = WaTor(kind, egg, en, FB=6, SB=12, SS=6, seed=42, stream=stream, shard=(rank, world))
            sim.exchange = WtExchange(sim)
            dist.barrier()
        else:
            sim = WaTor(kind, egg, en, FB=6, SB=12, SS=6, seed=42, stream=stream)
        step_fn = sim.step
        if world == 1:                     # one step replayed as a CUDA graph (no host launch overhead)
            sim.capture()
            step_fn = sim.graph.replay

        def per(k):
            for t in range(2):
                sim.heap.live_count_async(t, live[k, t], stream)
        ms = time_steps(step_fn, K, W, stream, per)
        lv = live.cpu().numpy()
        # visits of step k: 4 cell passes + 2 passes over the fish and sharks alive at its start
        starts = np.vstack([lv[:1] * 0 + lv[0], lv[:-1]])       # approx: counts at the previous step end
        visits = 4 * sim.W * sim.H * K + 2 * int(starts[:, 0].sum() + starts[:, 1].sum())   # this shard's
        visits, = reduce_over_ranks([float(visits)], "sum")
        ms, = reduce_over_ranks([ms], "max")
        cfg = {"workload": "wator (BASELINE configs[1]) 2048^2, FB6 SB12 SS6, seed 42",
               "parallelism": f"{world} row bands, NCCL P2P halo (4 exchanges per half step)" if world > 1
               else "1 GPU"}
        if world == 1:                     # the paper's static-allocation baseline, same start
            from paper_1810_11765_b200.wator import WaTorStatic
            base = WaTorStatic(kind, egg, en, FB=6, SB=12, SS=6, seed=42, stream=stream)
            bms = time_steps(lambda: base.run(1), K, W, stream)
            cfg["static_baseline"] = {"ms_per_step": bms, "dynamic_over_static": ms / bms,
                                      "what": "same rules on cell-indexed SOA arrays, no heap (dsr_wator_static_step)"}
    elif args.workload in ("gol", "gol16k", "gol16k-bits"):
        from paper_1810_11765_b200.gol import GameOfLife, NcclHaloExchange
        Wd = 64 if args.workload == "gol" else 16384
        a0 = I.gol_soup(Wd, Wd, 0.3 if Wd == 64 else 0.25, 1 if Wd == 64 else 42)
        if world > 1:                      # row bands + NCCL exchange of boundary masks
            sim = GameOfLife(a0, stream=stream, shard=(rank, world), bit_mirror=args.workload.endswith("bits"))
            sim.exchange = NcclHaloExchange(sim)
            dist.barrier()
        else:
            sim = GameOfLife(a0, stream=stream, bit_mirror=args.workload.endswith("bits"))
        step_fn = sim.generation
        if Wd == 64:                       # launch-bound: replay one generation as a CUDA graph
            sim.capture()
            step_fn = sim.graph.replay

        def per(k):
            for t in range(2):
                sim.heap.live_count_async(t, live[k, t], stream)
        ms = time_steps(step_fn, K, W, stream, per)
        lv = live.cpu().numpy()
        visits = 2 * int(lv[:, 0].sum() + lv[:, 1].sum())
        visits, = reduce_over_ranks([float(visits)], "sum")
        ms, = reduce_over_ranks([ms], "max")
        cfg = {"workload": f"gol {Wd}^2 torus (BASELINE configs[{0 if Wd == 64 else 3}])"
                           + (", alive-bit mirror variant" if args.workload.endswith("bits") else ""),
               "parallelism": f"{world} row bands, NCCL P2P halo masks" if world > 1 else "1 GPU"}
    else:
        from paper_1810_11765_b200.nbody import NBody
        st = I.nbody_init(65536, seed=7)
        # N > 1: id-range shards, S/V/target all-gathered over NCCL
        sim = NBody(st, merges=True, stream=stream, group=dist.group.WORLD if world > 1 else None,
                    **I.NBODY_PARAMS)

        def per(k):
            sim.heap.live_count_async(0, live[k, 0], stream)
        if world > 1:
            dist.barrier()
        ms = time_steps(sim.step, K, W, stream, per)
        lv = live.cpu().numpy()
        visits = 8 * int(lv[:, 0].sum())
        visits, = reduce_over_ranks([float(visits)], "sum")
        ms, = reduce_over_ranks([ms], "max")
        cfg = {"workload": "nbody with merging (BASELINE configs[2]) 65536 bodies", "pairs_per_step": 2 * 65536 ** 2,
               "pair_interactions_per_s": 2 * 65536 ** 2 / (ms * 1e-3),
               "parallelism": f"{world} id-range shards, NCCL all-gather of snapshot chunks" if world > 1 else "1 GPU"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = app_cpu_baseline(args.workload)
        except Exception as e:   # the line must still print
            cpu = {"value": None, "unit": "object-updates/s", "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}
    if rank == 0:
        if cpu is not None:
            cfg["cpu_baseline"] = cpu
        print(json.dumps({"metric": METRIC, "value": visits / K / (ms * 1e-3), "unit": "object-updates/s",
                          "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "strong", "dtype": "u32" if args.workload != "nbody" else "f32",
                          "data": "synthetic", "config": cfg}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def app_cpu_baseline(workload):
    """The oracle (plain C, one core) on a bounded prefix of the same app
    workload, in object-updates/s counted the way the GPU line counts them
    (the runs are identical, so the object counts are the same)."""
    import numpy as np
    from oracle import oracle as O
    from paper_1810_11765_b200 import inputs as I
    O.build()
    if workload == "wator":
        kind, egg, en = I.wator_init(2048, 2048, seed=42)
        S = 10
        t0 = time.perf_counter()
        _, _, _, c = O.wator_run(kind, egg, en, FB=6, SB=12, SS=6, seed=42, steps=S)
        t = time.perf_counter() - t0
        agents = [int((kind != 0).sum())] + [int(c[i, 0] + c[i, 1]) for i in range(S - 1)]
        visits = 4 * 2048 * 2048 * S + 2 * sum(agents)
        sample = f"first {S} steps of the 2048^2 run (object oracle), {t:.1f} s"
    elif workload in ("gol", "gol16k", "gol16k-bits"):
        Wd = 64 if workload == "gol" else 16384
        a0 = I.gol_soup(Wd, Wd, 0.3 if Wd == 64 else 0.25, 1 if Wd == 64 else 42)
        if Wd > 64:                  # bounded sample: one quadrant of the same soup, as its own torus
            a0 = np.ascontiguousarray(a0[:Wd // 2, :Wd // 2])
        G = 100 if Wd == 64 else 1
        t0 = time.perf_counter()
        O.gol_run(a0, G)
        t = time.perf_counter() - t0
        visits = 0
        a = a0
        for g in range(G):      # objects at each generation's start: alive + dead cells next to an alive one
            n = sum(np.roll(np.roll(a, dy, 0), dx, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)) - a
            visits += 2 * (int(a.sum()) + int(((a == 0) & (n > 0)).sum()))
            if g + 1 < G:
                a = O.life_dense(a, 1)
        sample = (f"first {G} generation(s) of the {a0.shape[0]}^2 " + ("run" if Wd == 64 else "quadrant of the same soup")
                  + f" (object oracle), {t:.1f} s")
    else:
        n = 32768                    # bounded sample: half the bodies (a quarter of the pairs)
        st = I.nbody_init(n, seed=7)
        t0 = time.perf_counter()
        O.nbody_run(st, merges=True, steps=1, **I.NBODY_PARAMS)
        t = time.perf_counter() - t0
        visits = 8 * n
        sample = f"one step of {n} bodies (oracle: fp32 state, fp64 arithmetic; {n * n / t:.3g} pairs/s), {t:.1f} s"
    return {"value": visits / t, "unit": "object-updates/s", "cores": 1, "kind": "oracle", "sample": sample}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload != "microbench":
        run_app(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
