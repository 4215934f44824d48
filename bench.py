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
    ap.add_argument("--workload", default="microbench", choices=["microbench", "wator", "gol", "gol16k", "gol16k-bits",
                                                                     "gol16k-tiled", "nbody"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-apps", action="store_true", help="skip the per-app block of the default line")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="sharded apps under torchrun: NCCL collectives, or peer memory (GoL: DSR_K_GOL_HALO_PUSH "
                         "into the neighbours' IPC-mapped halo buffers; N-body: the snapshot pass stores into "
                         "every rank's buffers)")
    ap.add_argument("--launch-list", action="store_true",
                    help="run only W + K microbench steps (for ncu launch lists) and print no bench line")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU work: exercise the launch / rank aggregation / JSON path (gloo; tests)")
    return ap.parse_args()


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def maybe_spawn(args):
    """--gpus N > 1 without a torchrun environment: re-launch this command
    under torch.distributed.run with N ranks on this node (127.0.0.1), so
    `python bench.py --gpus N` and the driver's torchrun launch are the same."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(ROOT / "bench.py"), *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(build_src):
    """Per-launch DRAM bytes (read + write), warp instructions and L2 atomic
    requests of the roofline kernels from committed `ncu --set full` summaries
    (profiles/<round>/ncu_summary.json) -- only those whose `build` (the
    library's source hash, recorded when they were captured) equals this
    library's; otherwise nothing (the counts would be stale)."""
    out = {}
    for p in sorted((ROOT / "profiles").glob("r*/ncu_summary.json")):
        try:
            rows = json.loads(p.read_text())
        except Exception:
            continue
        rows = [r for r in rows if build_src and build_src in r.get("build", "")]
        for key in ("k_mb_new_bulk", "k_mb_reduce"):
            for name, field in (("", "dram_bytes"), (":inst", "inst_executed"), (":atom", "l2_atom_alu_requests")):
                v = [r[field] for r in rows if key in r.get("kernel", "") and field in r]
                if v:
                    out[key + name] = sum(v) / len(v)
                    out[key + ":source"] = str(p.relative_to(ROOT))
    return out


def src_tag(info):
    """'src:<hash>' of a dsr_build_info() string."""
    for w in info.split():
        if w.startswith("src:"):
            return w
    return ""


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


def dist_init(n, backend=None):
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != n:
        raise SystemExit(f"bench.py --gpus {n} but WORLD_SIZE={world}")
    if torch.cuda.is_available() and backend != "gloo":
        torch.cuda.set_device(local)
    if world > 1:
        be = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(be)
        print(f"[bench] rank {rank}/{world} local {local} backend {be} (torch.distributed process group; "
              f"NCCL_DEBUG=INFO shows the communicator)", file=sys.stderr, flush=True)
    return rank, world, local


def reduce_over_ranks(vals, op, device=None):
    """Sum ("sum") or max ("max") of a list of floats over all ranks (identity
    without an initialised process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(vals)
    if device is None:
        device = "cuda" if dist.get_backend() == "nccl" else "cpu"
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
        "config": dict(CONFIG, n1=N1 // 4, n2=N2 // 4, full_workload={"n1": N1, "n2": N2},
                       sample="each step runs the microbench phases on a quarter of the workload "
                              "(n1 = 2^24, n2 = 2^23); object-updates/s is per object, so it compares "
                              "with the full-size line"),
        "cpu_baseline": {"value": v, "unit": "object-updates/s", "cores": 1, "kind": "oracle",
                         "sample": f"each step: the microbench phases on n1 = 2^24, n2 = 2^23 (a quarter of the "
                                   f"workload), oracle/ plain C single-threaded object store, {t:.2f} s/step"},
        "e2e": {"value": v, "unit": "object-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU leg
def mb_step_ms(mb, stream, K, W):
    """Device ms of one microbench step (K steps between events after W warm-up)."""
    import torch
    for _ in range(W):
        mb.step(stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K):
        mb.step(stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


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
    build_info = dsr.lib().dsr_build_info().decode()
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
    if args.launch_list:
        # only the step's own kernels (for `ncu --metrics gpu__time_duration.sum`
        # launch lists): K steps after the warm-up, no probe / variants / e2e / apps
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        assert mb.heap.poll_error() == dsr.OK
        if rank == 0:
            print(json.dumps({"launch_list_steps": args.steps, "warmup": args.warmup}), flush=True)
        return

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
    mb.step(stream=stream, stop=1)
    blocks.append(mb.heap.fragmentation(stream)[1])
    mb.heap.reset(stream)
    mb.step(stream=stream, stop=4)
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
    # dominant kernel: k_mb_new_bulk (device new + constructors, phases new1 / new4).
    # Algorithmic bytes = the constructed objects' fields + 16 B per block
    # initialised (type id + object bitmap), SURVEY §8(d) D5.
    per_type = lambda n: [(n + 1) // 2, n // 4 + (1 if n % 4 > 2 else 0), n // 4]   # [A,A,B,C][t&3]
    field_bytes = sum(c * s for c, s in zip(per_type(N1), sizes)) + sum(c * s for c, s in zip(per_type(N2), sizes))
    new_bytes = field_bytes + 16 * sum(int(b) for b in blocks[1])
    new_ms = phase_ms[1] + phase_ms[4]
    new_gbs = new_bytes / (new_ms * 1e-3) / 1e9
    shares = {p: v / ms for p, v in zip(["init", "new1", "reduce2", "free3", "new4", "reduce5", "drain6"], phase_ms)}
    traffic = ncu_traffic(src_tag(build_info))
    sm_mhz = clk.get("sm_mhz") or 1965.0

    # companions (untimed for the headline, timed the same way): the paper's per-thread device
    # new (one coalesced request per warp and type, Alg. 1) with and without the host-side
    # block reservation that round 1 used
    variants = {}
    if not args.no_apps:
        for name, kw in (("per_thread_new", dict(bulk=False)), ("per_thread_new_host_reserve", dict(bulk=False, reserve=True))):
            mv = Microbench(n1=N1, n2=N2, seed=SEED, stream=stream, **kw)
            variants[name] = {"ms_per_step": mb_step_ms(mv, stream, 3, 2)}
            assert mv.heap.poll_error() == dsr.OK
            del mv
            torch.cuda.empty_cache()

    # ---- e2e through the C ABI with HOST buffers: every step passes the host
    # (pinned) arrays of its 2^26 + 2^25 new objects' field values
    # (inputs.mb_fields, 1.61 GB) to dsr_launch(K_MB_NEW_BULK, in_host = 1),
    # which copies them into the heap's device staging buffers on its own copy
    # stream (overlapping the work already queued), and reads the 144-byte result back.
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
    del in1_h, in2_h

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

    apps = None
    if world == 1 and not args.no_apps:
        del mb
        torch.cuda.empty_cache()
        apps = app_block(stream, peak, peak_src, sm_mhz, want_cpu=not args.no_cpu_baseline)

    if rank == 0:
        inst = traffic.get("k_mb_new_bulk:inst")
        atom = traffic.get("k_mb_new_bulk:atom")
        line = {
            "metric": METRIC, "value": value, "unit": "object-updates/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": dict(CONFIG, heap_bytes=mb_heap_bytes(), caps=caps,
                           parallelism=f"{world} independent heaps (one per GPU)",
                           allocation="warp-cooperative bulk device new (K_MB_NEW_BULK, reading R-BULK); "
                                      "no host-side block reservation"),
            "allocs_per_s": (N1 + N2) * world / (new_ms * 1e-3),
            "frees_per_s": counts["frees"] * world / (sum(phase_ms[i] for i in (3, 6)) * 1e-3),
            "scan_gbs": scan_gbs,
            "phase_ms": dict(zip(["init", "new1", "reduce2", "free3", "new4", "reduce5", "drain6"], phase_ms)),
            "phase_share": shares,
            "fragmentation_after_phase4": frag5,
            "allocation_variants": variants,
            "roofline": {"bound": "hbm", "kernel": "k_mb_new_bulk (device new + constructors, 2 launches/step; "
                                                  f"{100 * new_ms / ms:.0f}% of the step)",
                         "achieved": new_gbs, "peak": peak, "unit": "GB/s", "frac": new_gbs / peak,
                         "traffic": traffic.get("k_mb_new_bulk"), "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": new_bytes / 2,
                         "traffic_source": traffic.get("k_mb_new_bulk:source"),
                         "note": "constructor writes (fields + block headers); the kernel is issue-bound on the "
                                 "workload's SplitMix64 field keys (roofline_issue)"},
            # the allocation kernel's warp instructions (committed ncu summary of THIS build, per new1
            # launch) / live new1 time, against 148 SMs x 4 schedulers x 1 warp-instruction/clk
            "roofline_issue": None if inst is None else {
                "bound": "issue", "kernel": "k_mb_new_bulk (phase new1 launch)",
                "achieved": inst / (phase_ms[1] * 1e-3) / 1e9,
                "peak": 148 * 4 * sm_mhz * 1e6 / 1e9, "unit": "G warp-inst/s",
                "frac": inst / (phase_ms[1] * 1e-3) / (148 * 4 * sm_mhz * 1e6),
                "inst_per_alloc": inst / N1, "source": traffic.get("k_mb_new_bulk:source")},
            "roofline_atomics": None if atom is None else {
                "bound": "l2_atomics", "kernel": "k_mb_new_bulk (phase new1 launch)",
                "achieved": atom / (phase_ms[1] * 1e-3) / 1e9, "peak": atom_peak / 1e9, "unit": "G atomics/s",
                "frac": atom / (phase_ms[1] * 1e-3) / atom_peak, "atomics_per_alloc": atom / N1,
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
            "apps": apps,
            "gpu_launches": launches,
            "clocks": clk,
            "build": build_info,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def mb_heap_bytes():
    return max(64 << 20, int((N1 + N2) * 24 * 2.0))


# ---------------------------------------------------------------- the other BASELINE configs (apps block)
def timed_steps(step, K, W, stream, after=None):
    """W untimed steps, then K steps each between its own pair of CUDA events on
    `stream`; after(k) runs between steps, outside the events (live counts).
    Returns the per-step device ms."""
    import torch
    for _ in range(W):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        if after is not None:
            after(k)
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def app_traffic(name, kernels=None):
    """DRAM bytes (read + write) per step of an app from the committed ncu
    summary profiles/<round>/ncu_<name>.json (one generation / step of the
    app's passes, scripts/gpu_ncu_apps.sh), only if it was captured from this
    library build (source hash); kernels: only those kernel names (per launch)."""
    if not name:
        return None
    from paper_1810_11765_b200 import dsr
    tag = src_tag(dsr.lib().dsr_build_info().decode())
    best = None
    for p in sorted((ROOT / "profiles").glob(f"r*/ncu_{name}.json")):
        try:
            rows = [r for r in json.loads(p.read_text()) if tag and tag in r.get("build", "")]
        except Exception:
            continue
        if kernels:
            rows = [r for r in rows if any(k in r.get("kernel", "") for k in kernels)]
        if rows:
            tot = sum(r.get("dram_bytes", 0.0) for r in rows)
            best = {"traffic": tot / len(rows) if kernels else tot,
                    "traffic_source": f"{p.relative_to(ROOT)} ({len(rows)} launches, "
                                      + ("per launch" if kernels else "one step") + ")"}
    return best


def full_length(step, n, stream, live_types, heap):
    """The BASELINE config's whole run (n steps from the initial state, which
    the caller just built): one pair of CUDA events around all n steps, the
    live counts of `live_types` recorded on the device after every step (tiny
    kernels, inside the events).  Returns (ms per step, live counts (n, k))."""
    import torch
    cnt = torch.zeros(n, len(live_types), dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for k in range(n):
        step()
        for j, t in enumerate(live_types):
            heap.live_count_async(t, cnt[k, j], stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, cnt.cpu().numpy()


def hbm_roofline(kernel, nbytes, ms, peak, peak_src, note, bound="hbm"):
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"bound": bound, "kernel": kernel, "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
            "algorithmic_bytes_per_step": nbytes, "peak_source": peak_src, "note": note}


def app_block(stream, peak, peak_src, sm_mhz, want_cpu=True):
    """BASELINE configs[0]-[3] on one GPU, each timed on the device (events
    around every step; live counts between steps, outside the events):
    object-updates/s, a roofline against MEASURED_PEAKS (SURVEY §8(d) D1-D4
    algorithmic work) and the oracle on a bounded sample."""
    import numpy as np
    import torch
    from paper_1810_11765_b200 import inputs as I
    out = {}
    live = torch.zeros(64, 3, dtype=torch.int64, device="cuda")

    def cpu_of(fn):
        if not want_cpu:
            return None
        try:
            return fn()
        except Exception as e:
            return {"value": None, "kind": "oracle", "cores": 1, "sample": f"failed: {e}"}

    # ---- GoL (configs[0] 64^2 x 100 gens; configs[3] 16384^2, handle grid and alive-bit mirror)
    from paper_1810_11765_b200.gol import GameOfLife
    # gol_16384: the prepare passes (the neighbour gathers) as cell-tiled do-alls
    # staging handle tiles in shared memory, the update passes on the block list
    # (DESIGN.md §6); gol_16384_blocklist: all four passes as the paper's
    # block-list do-all; gol_16384_bits: block list + the alive-bit mirror
    for name, Wd, K, Wu, bits, tiled in (("gol_64", 64, 100, 5, False, False),
                                         ("gol_16384", 16384, 4, 1, False, "prepare"),
                                         ("gol_16384_blocklist", 16384, 4, 1, False, False),
                                         ("gol_16384_bits", 16384, 4, 1, True, False)):
        a0 = I.gol_soup(Wd, Wd, 0.3 if Wd == 64 else 0.25, 1 if Wd == 64 else 42)
        sim = GameOfLife(a0, stream=stream, bit_mirror=bits, tiled=tiled)
        step = sim.generation
        if Wd == 64:
            sim.capture()
            step = sim.graph.replay
        cnt = torch.zeros(K, 2, dtype=torch.int64, device="cuda")

        def after(k, sim=sim, cnt=cnt):
            for t in range(2):
                sim.heap.live_count_async(t, cnt[k, t], stream)
        t = timed_steps(step, K, Wu, stream, after)
        lv = cnt.cpu().numpy()
        objs = lv.sum(axis=1)                                   # Alive + Candidate at each generation's start
        ms = sum(t) / K
        visits = 2 * int(objs.sum())                            # prepare + update visit per object
        nbytes = 88 * float(objs.mean())                        # ~88 B per object and generation
        out[name] = {
            "config": f"BASELINE configs[{0 if Wd == 64 else 3}]: {Wd}^2 torus, Bernoulli("
                      f"{0.3 if Wd == 64 else 0.25}) soup" + (", alive-bit mirror variant" if bits else "")
                      + (", prepare passes as cell-tiled do-alls (objects enumerated through the handle grid, "
                         "(8+2) x (128+2) handle tiles in shared memory), update passes on the block list" if tiled
                         else (", all passes on the block list" if Wd > 64 and not bits else ""))
                      + (", one generation replayed as a CUDA graph" if Wd == 64 else ""),
            "value": visits / (sum(t) * 1e-3), "unit": "object-updates/s", "ms_per_step": ms, "steps": K,
            "objects_per_step": float(objs.mean()),
            "roofline": hbm_roofline("whole generation (4 do-alls + prologues)", nbytes, ms, peak, peak_src,
                                     "launch/latency-bound: 4 do-alls over <= 4 K objects, no roofline target "
                                     "(SURVEY D1)" if Wd == 64 else
                                     "88 B/object/gen (own fields + 8 neighbour handles + update), SURVEY D4; "
                                     "the neighbour gathers are scattered (objects sit in blocks in allocation, "
                                     "not grid, order: P:794)" + ("; this variant reads a 1-bit mirror instead of "
                                                                  "the 8 handles, same algorithmic definition" if bits else ""),
                                     bound="latency" if Wd == 64 else "hbm"),
        }
        if name == "gol_16384":
            # the whole BASELINE run: 1000 generations from the soup (the density falls
            # from 0.25 to a few %, so late generations are much cheaper than the first)
            del sim
            torch.cuda.empty_cache()
            sim = GameOfLife(a0, stream=stream, bit_mirror=bits, tiled=tiled)
            init = sim.heap.live_count(0, stream) + sim.heap.live_count(1, stream)
            fms, flv = full_length(sim.generation, 1000, stream, (0, 1), sim.heap)
            visits = 2 * (init + int(flv[:-1].sum()))            # objects at the start of each generation
            out[name]["full_length"] = {
                "generations": 1000, "ms_per_step": fms, "value": visits / (1000 * fms * 1e-3),
                "unit": "object-updates/s", "objects_first_last": [init, int(flv[-1].sum())],
                "note": "all 1000 generations of configs[3] timed as one region (live counts recorded on the "
                        "device each generation); object-updates = prepare + update visit of every object"}
        tr = app_traffic({"gol_16384": "gol16k-tiled", "gol_16384_blocklist": "gol16k",
                          "gol_16384_bits": "gol16k-bits"}.get(name))
        if tr:
            out[name]["roofline"].update(tr)
        del sim
        torch.cuda.empty_cache()
        if name != "gol_64" and name != "gol_16384":
            continue
        from paper_1810_11765_b200.gol import GameOfLifeStatic
        base = GameOfLifeStatic(a0, stream=stream)
        tb = timed_steps(lambda: base.run(1), K, Wu, stream)
        out[name]["static_baseline"] = {"ms_per_step": sum(tb) / K, "dynamic_over_static": ms / (sum(tb) / K),
                                        "what": "B3/S23 on a u8 cell grid, no objects (P:763, dsr_gol_static_step)"}
        del base

        def gol_cpu(Wd=Wd):
            from oracle import oracle as O
            O.build()
            b = I.gol_soup(Wd, Wd, 0.3 if Wd == 64 else 0.25, 1 if Wd == 64 else 42)
            if Wd > 64:
                b = np.ascontiguousarray(b[:4096, :4096])     # bounded sample: a 4096^2 corner as its own torus
            G = 100 if Wd == 64 else 1
            t0 = time.perf_counter()
            O.gol_run(b, G)
            dt = time.perf_counter() - t0
            vis, a = 0, b
            for _ in range(G):
                n = sum(np.roll(np.roll(a, dy, 0), dx, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)) - a
                vis += 2 * (int(a.sum()) + int(((a == 0) & (n > 0)).sum()))
                a = O.life_dense(a, 1)
            return {"value": vis / dt, "unit": "object-updates/s", "cores": 1, "kind": "oracle",
                    "sample": f"{G} generation(s) of " + (f"the {Wd}^2 run" if Wd == 64 else
                                                         "a 4096^2 corner of the same soup (own torus)")
                              + f", object oracle, {dt:.2f} s"}
        out[name]["cpu_baseline"] = cpu_of(gol_cpu)

    # ---- Wa-Tor 2048^2 (configs[1]); the static SOA baseline beside it
    from paper_1810_11765_b200.wator import WaTor, WaTorStatic
    kind, egg, en = I.wator_init(2048, 2048, seed=42)
    sim = WaTor(kind, egg, en, FB=6, SB=12, SS=6, seed=42, stream=stream)
    sim.capture()
    K = 40
    cnt = torch.zeros(K, 2, dtype=torch.int64, device="cuda")

    def after(k):
        for t in range(2):
            sim.heap.live_count_async(t, cnt[k, t], stream)
    t = timed_steps(sim.graph.replay, K, 5, stream, after)
    agents = cnt.cpu().numpy().sum(axis=1)
    cells = 2048 * 2048
    ms = sum(t) / K
    visits = 4 * cells * K + 2 * int(agents.sum())
    nbytes = 20 * cells + 100 * float(agents.mean())
    base = WaTorStatic(kind, egg, en, FB=6, SB=12, SS=6, seed=42, stream=stream)
    tb = timed_steps(lambda: base.run(1), K, 5, stream)
    out["wator_2048"] = {
        "config": "BASELINE configs[1]: 2048^2 torus, FB 6 SB 12 SS 6, seed 42; one step (8 do-alls) replayed "
                  "as a CUDA graph",
        "value": visits / (sum(t) * 1e-3), "unit": "object-updates/s", "ms_per_step": ms, "steps": K,
        "agents_per_step": float(agents.mean()),
        "roofline": hbm_roofline("whole step (8 do-alls + prologues)", nbytes, ms, peak, peak_src,
                                 "SURVEY D2: 2 x 5 B req clears + 2 x 5 B decides per cell + ~100 B per agent; "
                                 "working set ~80 MB is L2-resident (126 MB), so HBM is not the bound"),
        "static_baseline": {"ms_per_step": sum(tb) / K, "dynamic_over_static": ms / (sum(tb) / K),
                            "what": "same rules on cell-indexed SOA arrays, no heap (P:763, dsr_wator_static_step)"},
        "fragmentation": sim.heap.fragmentation()[0],
    }
    tr = app_traffic("wator")
    if tr:
        out["wator_2048"]["roofline"].update(tr)
    del sim, base
    torch.cuda.empty_cache()
    sim = WaTor(kind, egg, en, FB=6, SB=12, SS=6, seed=42, stream=stream)
    sim.capture()                                                # runs step 1 (the warm-up of the capture)
    ag1 = sim.heap.live_count(0, stream) + sim.heap.live_count(1, stream)
    fms, flv = full_length(sim.graph.replay, 499, stream, (0, 1), sim.heap)
    last = [int(flv[-1, 0]), int(flv[-1, 1])]
    gold = ROOT / "tests" / "golden" / "wator2048_500steps.npz"
    want = [int(v) for v in np.load(gold)["counters"][-1, :2]] if gold.exists() else None
    out["wator_2048"]["full_length"] = {
        "steps": 500, "timed_steps": 499, "ms_per_step": fms,
        "value": (4 * cells * 499 + 2 * (ag1 + int(flv[:-1].sum()))) / (499 * fms * 1e-3),
        "unit": "object-updates/s", "fish_sharks_after_500": last, "equals_oracle_golden": last == want,
        "note": "configs[1]: step 1 runs while the step's CUDA graph is captured, steps 2-500 are graph replays "
                "timed as one region; the final populations are checked against the oracle's "
                "(tests/golden/wator2048_500steps.npz)"}
    del sim
    torch.cuda.empty_cache()

    def wator_cpu():
        from oracle import oracle as O
        O.build()
        S = 2
        t0 = time.perf_counter()
        _, _, _, c = O.wator_run(kind, egg, en, FB=6, SB=12, SS=6, seed=42, steps=S)
        dt = time.perf_counter() - t0
        ag = [int((kind != 0).sum())] + [int(c[i, 0] + c[i, 1]) for i in range(S - 1)]
        return {"value": (4 * cells * S + 2 * sum(ag)) / dt, "unit": "object-updates/s", "cores": 1,
                "kind": "oracle", "sample": f"first {S} steps of the 2048^2 run (object oracle), {dt:.2f} s"}
    out["wator_2048"]["cpu_baseline"] = cpu_of(wator_cpu)

    # ---- N-body 65,536 bodies with merging (configs[2]); the force pass against the FP32 pipe
    from paper_1810_11765_b200 import dsr
    from paper_1810_11765_b200.nbody import NBody
    st = I.nbody_init(65536, seed=7)
    sim = NBody(st, merges=True, stream=stream, **I.NBODY_PARAMS)
    K = 10
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K + 3)]
    kk = [0]

    def nb_step():
        e = fev[kk[0]]
        sim.p_snapshot(stream)
        e[0].record(stream)
        sim.heap.parallel_do(0, dsr.M_NB_FORCE, sim.args, stream)
        e[1].record(stream)
        sim.heap.parallel_do(0, dsr.M_NB_MOVE, sim.args, stream)
        sim.p_snapshot(stream)
        sim.p_merge_search(stream)
        sim.p_claim_absorb_delete(stream)
        kk[0] += 1
    cnt = torch.zeros(K, 1, dtype=torch.int64, device="cuda")

    def after(k):
        sim.heap.live_count_async(0, cnt[k, 0], stream)
    t = timed_steps(nb_step, K, 3, stream, after)
    lv = cnt.cpu().numpy()[:, 0]
    ms = sum(t) / K
    force_ms = sum(fev[3 + k][0].elapsed_time(fev[3 + k][1]) for k in range(K)) / K
    pairs = float((lv.astype(np.float64) ** 2).mean())          # the force pass: every pair of existing bodies
    fp32_peak = 148 * 128 * sm_mhz * 1e6                        # FP32 lanes x SM clock
    ops = 9.0 * pairs                                           # 9 FP32 ops per pair + 1 MUFU.RSQ
    out["nbody_65536"] = {
        "config": "BASELINE configs[2]: 65,536 fp32 bodies with merging, seed 7, inputs.NBODY_PARAMS",
        "value": 8 * float(lv.sum()) / (sum(t) * 1e-3), "unit": "object-updates/s", "ms_per_step": ms, "steps": K,
        "pair_interactions_per_s": 2 * pairs / (ms * 1e-3),
        "roofline": {"bound": "alu", "kernel": f"k_nb_force_part (compute_force, device_do all-pairs; "
                                               f"{100 * force_ms / ms:.0f}% of the step)",
                     "achieved": ops / (force_ms * 1e-3) / 1e12, "peak": fp32_peak / 1e12, "unit": "T FP32 op/s",
                     "frac": ops / (force_ms * 1e-3) / fp32_peak, "force_ms": force_ms,
                     "peak_source": "148 SMs x 128 FP32 lanes x sampled SM clock (B200_PROFILING.md unit counts)",
                     "note": "9 FP32 ops per pair (2 FADD, 2 FFMA for r^2, 3 FMUL, 2 FFMA accumulate) on packed "
                             "f32x2 pairs, over the pairs of existing bodies (the live list); the snapshot is "
                             "SMEM/L2-resident"},
    }
    tr = app_traffic("nbody", kernels=("k_nb_force_part",))
    if tr:
        out["nbody_65536"]["roofline"].update(tr)
    del sim
    torch.cuda.empty_cache()
    sim = NBody(st, merges=True, stream=stream, **I.NBODY_PARAMS)
    fms, flv = full_length(lambda: sim.step(stream), 1000, stream, (0,), sim.heap)
    out["nbody_65536"]["full_length"] = {
        "steps": 1000, "ms_per_step": fms,
        "value": 8 * (65536 + float(flv[:-1, 0].sum())) / (1000 * fms * 1e-3), "unit": "object-updates/s",
        "bodies_last": int(flv[-1, 0]),
        "note": "all 1000 steps of configs[2] timed as one region (bodies merge: 65,536 -> ~18 k)"}
    del sim
    torch.cuda.empty_cache()
    from paper_1810_11765_b200.nbody import NBodyStatic
    base = NBodyStatic(st, merges=True, stream=stream, **I.NBODY_PARAMS)
    tb = timed_steps(lambda: base.run(1), K, 3, stream)
    out["nbody_65536"]["static_baseline"] = {"ms_per_step": sum(tb) / K, "dynamic_over_static": ms / (sum(tb) / K),
                                             "what": "the same passes on id-indexed SOA arrays, no heap (P:763, "
                                                     "dsr_nbody_static_step)"}
    del base

    def nbody_cpu():
        from oracle import oracle as O
        O.build()
        n = 8192
        s2 = I.nbody_init(n, seed=7)
        t0 = time.perf_counter()
        O.nbody_run(s2, merges=True, steps=1, **I.NBODY_PARAMS)
        dt = time.perf_counter() - t0
        return {"value": 8 * n / dt, "unit": "object-updates/s", "cores": 1, "kind": "oracle",
                "sample": f"one step of {n} bodies (fp32 state, fp64 arithmetic; {2 * n * n / dt:.3g} pairs/s), "
                          f"{dt:.2f} s"}
    out["nbody_65536"]["cpu_baseline"] = cpu_of(nbody_cpu)
    return out


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
    if world > 1 and args.workload not in ("nbody", "gol16k", "gol16k-bits", "gol16k-tiled", "wator"):
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
    elif args.workload in ("gol", "gol16k", "gol16k-bits", "gol16k-tiled"):
        from paper_1810_11765_b200.gol import GameOfLife, NcclHaloExchange
        Wd = 64 if args.workload == "gol" else 16384
        a0 = I.gol_soup(Wd, Wd, 0.3 if Wd == 64 else 0.25, 1 if Wd == 64 else 42)
        if world > 1:                      # row bands + an exchange of boundary masks
            peer = args.exchange == "peer"
            sim = GameOfLife(a0, stream=stream, shard=(rank, world), bit_mirror=args.workload.endswith("bits"),
                             tiled=args.workload.endswith("tiled") and "prepare", peer=peer)
            if peer:                       # the neighbours' halo buffers mapped over NVLink (CUDA IPC)
                from paper_1810_11765_b200.gol import PeerHalo
                sim.peer_halo = PeerHalo(sim)
            else:
                sim.exchange = NcclHaloExchange(sim)
            dist.barrier()
        else:
            sim = GameOfLife(a0, stream=stream, bit_mirror=args.workload.endswith("bits"),
                             tiled=args.workload.endswith("tiled") and "prepare")
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
                           + (", alive-bit mirror variant" if args.workload.endswith("bits") else "")
                           + (", cell-tiled prepare passes" if args.workload.endswith("tiled") else ""),
               "parallelism": (f"{world} row bands, " + ("peer-memory push of the halo masks over NVLink"
                                                          if args.exchange == "peer" else "NCCL P2P halo masks"))
               if world > 1 else "1 GPU"}
    else:
        from paper_1810_11765_b200.nbody import NBody
        st = I.nbody_init(65536, seed=7)
        # N > 1: id-range shards, S/V/target all-gathered over NCCL, or (--exchange peer) stored by the
        # snapshot pass straight into every rank's IPC-mapped buffers
        sim = NBody(st, merges=True, stream=stream, group=dist.group.WORLD if world > 1 else None,
                    peer=args.exchange == "peer", **I.NBODY_PARAMS)
        if sim.peer:
            from paper_1810_11765_b200.nbody import NBodyPeer
            sim.peer_map = NBodyPeer(sim)

        def per(k):
            sim.heap.live_count_async(0, live[k, 0], stream)
        if world > 1:
            dist.barrier()
        ms = time_steps(sim.step, K, W, stream, per)
        lv = live.cpu().numpy()
        visits = 8 * int(lv[:, 0].sum())
        visits, = reduce_over_ranks([float(visits)], "sum")
        ms, = reduce_over_ranks([ms], "max")
        tot_live = reduce_over_ranks([float(v) for v in lv[:, 0]], "sum")     # bodies in existence per step
        pairs = 2 * float(np.mean(np.square(tot_live)))                       # force + merge pass pairs
        cfg = {"workload": "nbody with merging (BASELINE configs[2]) 65536 bodies", "pairs_per_step": pairs,
               "pair_interactions_per_s": pairs / (ms * 1e-3),
               "parallelism": (f"{world} id-range shards, " + ("snapshot / target rows stored into every "
                                                               "rank's memory over NVLink (peer mode)"
                                                               if args.exchange == "peer"
                                                               else "NCCL all-gather of snapshot chunks"))
               if world > 1 else "1 GPU"}
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


def run_dry(args):
    """--dry-run: the multi-rank plumbing without a GPU (gloo): every rank
    'processes' N1 + N2 objects in (1 + rank) ms; rank 0 prints the line with
    the summed work and the max-over-ranks time (tests/test_multiproc_cpu.py)."""
    import torch.distributed as dist
    rank, world, _ = dist_init(args.gpus, backend="gloo")
    work, = reduce_over_ranks([float(N1 + N2)], "sum", device="cpu")
    ms, = reduce_over_ranks([1.0 + rank], "max", device="cpu")
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": work / (ms * 1e-3), "unit": "object-updates/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "weak", "dry_run": True, "config": CONFIG}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    maybe_spawn(args)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.workload != "microbench":
        run_app(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
