"""world_size-2 gloo tests (CPU) of the multi-GPU host logic: the id-range
partition, the all-gather exchange of id-indexed arrays used by the sharded
N-body, and bench.py's max-over-ranks / sum-over-ranks aggregation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _exchange(rank, world):
    from paper_1810_11765_b200.nbody import Exchange, id_range
    n = 64
    lo, hi = id_range(n, world, rank)
    S = torch.zeros(n, 4)
    S[lo:hi] = torch.arange(lo, hi, dtype=torch.float32)[:, None] * torch.tensor([1.0, 2.0, 3.0, 0.0])
    tgt = torch.full((n,), -1, dtype=torch.int32)
    tgt[lo:hi] = torch.arange(lo, hi, dtype=torch.int32) * 7 % n
    x = Exchange(dist.group.WORLD)
    x.all_gather_rows(S, lo, hi)
    x.all_gather_rows(tgt, lo, hi)
    return S.numpy(), tgt.numpy(), (lo, hi)


def test_id_range_partition_and_exchange():
    out = run_world(_exchange, 2)
    n = 64
    want_S = np.arange(n, dtype=np.float32)[:, None] * np.array([1, 2, 3, 0], np.float32)
    want_t = (np.arange(n) * 7 % n).astype(np.int32)
    ranges = sorted(v[2] for v in out.values())
    assert ranges == [(0, 32), (32, 64)]
    for S, t, _ in out.values():
        assert np.array_equal(S, want_S) and np.array_equal(t, want_t)


def _aggregate(rank, world):
    import bench
    ms = [3.0, 5.0][rank]
    work = [100.0, 200.0][rank]
    tot, = bench.reduce_over_ranks([work], "sum", device="cpu")
    mx, = bench.reduce_over_ranks([ms], "max", device="cpu")
    return tot, mx


def test_bench_aggregation_max_time_sum_work():
    out = run_world(_aggregate, 2)
    for tot, mx in out.values():
        assert tot == 300.0 and mx == 5.0


def test_id_range_rejects_uneven():
    from paper_1810_11765_b200.nbody import id_range
    with pytest.raises(ValueError):
        id_range(10, 3, 0)


class _FakeGol:
    def __init__(self, rank, W):
        self.W = W
        self.halo = torch.zeros(4 * W, dtype=torch.uint8)
        self.halo[0:W] = 10 * rank + 1          # "my first row"
        self.halo[W:2 * W] = 10 * rank + 2      # "my last row"


def _gol_halo(rank, world):
    from paper_1810_11765_b200.gol import NcclHaloExchange, row_range
    sim = _FakeGol(rank, 8)
    NcclHaloExchange(sim)()
    return sim.halo.numpy().copy(), row_range(48, world, rank)


@pytest.mark.parametrize("world", [2, 3])
def test_gol_halo_exchange_routes_rows(world):
    """Top ghost row <- the upper shard's last row; bottom ghost row <- the
    lower shard's first row (torus of ranks), also when up == down (2 ranks)."""
    out = run_world(_gol_halo, world)
    W = 8
    for r, (h, band) in out.items():
        up, down = (r - 1) % world, (r + 1) % world
        assert (h[2 * W:3 * W] == 10 * up + 2).all()
        assert (h[3 * W:4 * W] == 10 * down + 1).all()
        assert band == (r * 48 // world, (r + 1) * 48 // world)


class _FakeWaTor:
    def __init__(self, rank, W):
        from paper_1810_11765_b200 import dsr
        self.W = W
        self.halo_layout = dsr.wt_halo_layout(W)
        self.halo = torch.zeros(self.halo_layout["bytes"], dtype=torch.uint8)
        for seg in ("req", "grant", "occ", "mig"):
            o, i, n = self.halo_layout[seg]
            self.halo[o:o + n] = 10 * rank + 1           # side 0: towards the shard above
            self.halo[o + n:o + 2 * n] = 10 * rank + 2   # side 1: towards the shard below


def _wt_halo(rank, world):
    from paper_1810_11765_b200.wator import NcclHaloExchange
    sim = _FakeWaTor(rank, 8)
    x = NcclHaloExchange(sim)
    for seg in ("req", "grant", "mig", "occ"):
        x(seg)
    return sim.halo.numpy().copy()


@pytest.mark.parametrize("world", [2, 3])
def test_wator_halo_exchange_routes_segments(world):
    """in[0] <- the upper shard's side-1 out, in[1] <- the lower shard's side-0
    out, for every segment (the migrant records are 12 B per column)."""
    from paper_1810_11765_b200 import dsr
    out = run_world(_wt_halo, world)
    L = dsr.wt_halo_layout(8)
    for r, h in out.items():
        up, down = (r - 1) % world, (r + 1) % world
        for seg in ("req", "grant", "occ", "mig"):
            o, i, n = L[seg]
            assert (h[i:i + n] == 10 * up + 2).all(), seg
            assert (h[i + n:i + 2 * n] == 10 * down + 1).all(), seg
            assert (h[o:o + n] == 10 * r + 1).all()              # out segments untouched


def test_bench_self_spawns_ranks_dry_run():
    """`python bench.py --gpus 2` (no torchrun environment) re-launches itself
    under torch.distributed.run with two ranks; the dry run (gloo, no GPU work)
    goes through the same rank aggregation: n_gpus = 2, work summed over the
    ranks, time = the max over ranks (1 + rank ms)."""
    import json
    import os
    import subprocess
    import sys
    from conftest import ROOT
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                     # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"]
    assert d["ms_per_step"] == 2.0
    assert d["value"] == 2 * ((1 << 26) + (1 << 25)) / 2e-3
