"""GPU parity of the Game of Life workload (BASELINE configs[0] / [3]) against
the oracle: canonical (cell, kind, is_new, action) records bit-exact every
generation at 64x64, alive bitmaps against the oracle's dense Life at larger
sizes, and the heap invariants after the run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1810_11765_b200 import build, gol
    build.build()
    return gol


@pytest.mark.parametrize("name", ["glider", "blinker", "soup1", "soup2", "soup3"])
def test_gol_64_every_generation_bit_exact(G, O, name):
    from paper_1810_11765_b200 import inputs as I
    a0 = I.gol_pattern(name) if not name.startswith("soup") else I.gol_soup(64, 64, 0.3, int(name[-1]))
    _, want = O.gol_run(a0, 100, dump=True)
    g = G.GameOfLife(a0)
    for gen in range(100):
        g.generation()
        got = g.records()
        assert np.array_equal(got, want[gen]), f"generation {gen + 1}"
    assert g.heap.poll_error() == 0
    assert g.heap.check_invariants() == 0


@pytest.mark.parametrize("W,H,p,seed,gens", [(37, 23, 0.4, 4, 60), (3, 3, 0.5, 6, 10), (512, 384, 0.25, 7, 50)])
def test_gol_ragged_sizes_against_dense_life(G, O, W, H, p, seed, gens):
    from paper_1810_11765_b200 import inputs as I
    a0 = I.gol_soup(W, H, p, seed)
    g = G.GameOfLife(a0)
    g.run(gens)
    assert np.array_equal(g.alive(), O.life_dense(a0, gens))
    assert g.heap.check_invariants() == 0


def test_gol_tiny_heap_forces_block_reuse(G, O):
    """A heap barely larger than the live set: blocks are freed and re-typed
    every generation (Alive <-> Candidate), exercising invalidation and rollback."""
    from paper_1810_11765_b200 import inputs as I
    a0 = I.gol_soup(64, 64, 0.3, 9)
    g = G.GameOfLife(a0, heap_bytes=600_000)
    g.run(100)
    assert g.heap.poll_error() == 0
    assert np.array_equal(g.alive(), O.life_dense(a0, 100))
    assert g.heap.check_invariants() == 0


@pytest.mark.slow
def test_gol_16384_sampled_against_dense(G, O):
    """BASELINE configs[3] size (16384^2, p = 0.25) for 3 generations: the
    oracle's dense Life runs on 9 sampled 256x256 windows whose 3-generation
    light cone is included (border of 3 cells)."""
    from paper_1810_11765_b200 import inputs as I
    W = H = 16384
    a0 = I.gol_soup(W, H, 0.25, 42)
    g = G.GameOfLife(a0)
    gens = 3
    g.run(gens)
    got = g.alive()
    rng = np.random.default_rng(0)
    for _ in range(9):
        y, x = int(rng.integers(0, H - 300)), int(rng.integers(0, W - 300))
        win = a0[y:y + 262, x:x + 262]
        want = O.life_dense(np.ascontiguousarray(win), gens)[3:259, 3:259]   # torus wrap only hits the border
        assert np.array_equal(got[y + 3:y + 259, x + 3:x + 259], want)
    assert g.heap.check_invariants() == 0


def test_gol_cuda_graph_replay(G, O):
    """One generation captured as a CUDA graph (device-side R count, no host
    sync inside a do-all) and replayed: same result as eager launches."""
    from paper_1810_11765_b200 import inputs as I
    a0 = I.gol_soup(64, 64, 0.3, 2)
    g = G.GameOfLife(a0)
    g.capture()                      # executes 1 generation (warm-up) + captures one
    g.run_graph(99)
    torch.cuda.synchronize()
    assert g.gen == 100
    assert np.array_equal(g.alive(), O.life_dense(a0, 100))
    assert g.heap.check_invariants() == 0


def test_gol_empty_grid_and_empty_passes(G, O):
    """Degenerate inputs: an empty grid has no objects; every do-all visits
    nothing and the heap stays empty."""
    import numpy as np
    g = G.GameOfLife(np.zeros((32, 48), np.uint8))
    g.run(3)
    assert g.alive().sum() == 0
    assert g.heap.live_count(0) == 0 and g.heap.live_count(1) == 0
    assert g.heap.check_invariants() == 0


@pytest.mark.parametrize("P,W,H,gens", [(1, 64, 64, 60), (2, 64, 64, 60), (4, 48, 40, 80), (8, 128, 64, 30)])
def test_gol_row_shards_loopback_equal_dense(G, O, P, W, H, gens):
    """Row-band sharding with ghost rows and one mask exchange per generation
    (P heaps on one GPU, messages as device copies) gives dense Life exactly."""
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLifeLoopback
    a0 = I.gol_soup(W, H, 0.3, P + 20)
    lb = GameOfLifeLoopback(a0, P)
    lb.run(gens)
    assert np.array_equal(lb.alive(), O.life_dense(a0, gens))
    for s in lb.shards:
        assert s.heap.check_invariants() == 0


@pytest.mark.parametrize("P,W,H,gens,tiled", [(1, 64, 64, 60, False), (2, 64, 64, 60, False),
                                              (3, 96, 48, 70, False), (4, 200, 64, 40, "prepare")])
def test_gol_peer_memory_exchange_equal_dense(G, O, P, W, H, gens, tiled):
    """The peer-memory halo exchange (DSR_K_GOL_HALO_PUSH stores each shard's
    boundary masks straight into its neighbours' halo buffers and sets their
    flags; DSR_K_GOL_HALO_APPLY waits on its own flags and reads the
    generation-parity slot): P heaps on one GPU exchanging through each
    other's device memory, no host copies, give dense Life every generation
    (P = 1: a shard is its own neighbour across the torus seam)."""
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLifeLoopback
    a0 = I.gol_soup(W, H, 0.3, P + 40)
    lb = GameOfLifeLoopback(a0, P, peer=True, tiled=tiled)
    a = a0
    for g in range(gens):
        lb.generation()
        a = O.life_dense(a, 1)
        if g % 10 == 9 or g == gens - 1:
            assert np.array_equal(lb.alive(), a), g
    for s in lb.shards:
        assert s.heap.check_invariants() == 0


def test_gol_peer_memory_exchange_two_processes(G, O):
    """Two processes (one shard each) map each other's halo buffers through
    CUDA IPC (handles all-gathered over gloo) and exchange only through that
    memory -- the multi-GPU path, here with both processes on one GPU."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29000 + os.getpid() % 1000),
           str(root / "tests" / "peer_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=str(root))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "PEER OK" in r.stdout, r.stdout[-3000:]


def test_gol_glider_crosses_shard_boundaries(G, O):
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLifeLoopback
    a0 = I.gol_pattern("glider")
    lb = GameOfLifeLoopback(a0, 4)                 # bands of 16 rows: the glider crosses all of them
    lb.run(4 * 64)
    assert np.array_equal(lb.alive(), a0)


@pytest.mark.parametrize("name", ["glider", "soup1"])
def test_gol_bit_mirror_variant_bit_exact(G, O, name):
    """The alive-bit mirror variant (prepare passes count neighbours from a
    1-bit-per-cell grid) yields the same records every generation."""
    from paper_1810_11765_b200 import inputs as I
    a0 = I.gol_pattern(name) if name == "glider" else I.gol_soup(64, 64, 0.3, 1)
    _, want = O.gol_run(a0, 60, dump=True)
    g = G.GameOfLife(a0, bit_mirror=True)
    for gen in range(60):
        g.generation()
        assert np.array_equal(g.records(), want[gen]), f"generation {gen + 1}"
    bits = g.bits.cpu().numpy().view(np.uint32)
    P = (64 + 31) // 32
    alive = np.array([[(bits[y * P + x // 32] >> (x % 32)) & 1 for x in range(64)] for y in range(64)], np.uint8)
    assert np.array_equal(alive, g.alive())                      # the mirror equals the object state
    assert g.heap.check_invariants() == 0


@pytest.mark.parametrize("W,H,P", [(45, 37, 1), (33, 40, 4), (31, 16, 2), (100, 64, 8)])
def test_gol_bit_mirror_ragged_and_sharded(G, O, W, H, P):
    """Widths that are not multiples of 32 (the x-1..x+1 window straddles
    words and the torus seam), alone and in row-band shards."""
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLifeLoopback
    a0 = I.gol_soup(W, H, 0.35, W + H)
    if H % P == 0 and P > 1:
        sim = GameOfLifeLoopback(a0, P, bit_mirror=True)
    else:
        sim = G.GameOfLife(a0, bit_mirror=True)
    sim.run(40)
    assert np.array_equal(sim.alive(), O.life_dense(a0, 40))


@pytest.mark.slow
def test_gol_16384_row_shards_equal_single_heap_and_dense(G, O):
    """BASELINE configs[3] as it is sharded at 8 GPUs: 8 row-band heaps of
    2048 rows (loopback exchange on one GPU) for 3 generations equal the
    single-heap GPU run everywhere and the oracle's dense Life on sampled
    windows, including windows that straddle band boundaries."""
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLifeLoopback
    W = H = 16384
    a0 = I.gol_soup(W, H, 0.25, 42)
    gens = 3
    lb = GameOfLifeLoopback(a0, 8)
    lb.run(gens)
    got = lb.alive()
    for s in lb.shards:
        assert s.heap.check_invariants() == 0
    del lb
    torch.cuda.empty_cache()
    g = G.GameOfLife(a0)
    g.run(gens)
    assert np.array_equal(got, g.alive())
    del g
    rng = np.random.default_rng(1)
    for y in [2048 - 131, 4096 - 131, int(rng.integers(0, H - 300)), 14336 - 131]:   # windows stay inside the grid
        x = int(rng.integers(0, W - 300))
        win = a0[y:y + 262, x:x + 262]
        want = O.life_dense(np.ascontiguousarray(win), gens)[3:259, 3:259]
        assert np.array_equal(got[y + 3:y + 259, x + 3:x + 259], want)


# ------------------------------------------------------------------ cell-tiled do-alls
@pytest.mark.parametrize("tiled", ["prepare", "all"])
@pytest.mark.parametrize("name", ["glider", "blinker", "soup1", "soup2"])
def test_gol_tiled_every_generation_bit_exact(G, O, name, tiled):
    """The cell-tiled passes (objects enumerated through the cell grid,
    neighbour handles staged in shared memory) give the oracle's records
    every generation, like the block-list passes."""
    from paper_1810_11765_b200 import inputs as I
    a0 = I.gol_pattern(name) if not name.startswith("soup") else I.gol_soup(64, 64, 0.3, int(name[-1]))
    _, want = O.gol_run(a0, 100, dump=True)
    g = G.GameOfLife(a0, tiled=tiled)
    for gen in range(100):
        g.generation()
        assert np.array_equal(g.records(), want[gen]), f"generation {gen + 1}"
    assert g.heap.poll_error() == 0
    assert g.heap.check_invariants() == 0


@pytest.mark.parametrize("tiled", ["prepare", "all"])
@pytest.mark.parametrize("W,H,p,seed,gens", [(37, 23, 0.4, 4, 60), (3, 3, 0.5, 6, 10), (129, 9, 0.3, 5, 40),
                                             (513, 385, 0.25, 7, 50), (128, 8, 0.35, 8, 30)])
def test_gol_tiled_ragged_sizes_against_dense_life(G, O, W, H, p, seed, gens, tiled):
    """Sizes that are not multiples of the 8 x 128 tile (ragged last tile row
    and column, torus wrap across tile edges) and the exact-tile case."""
    from paper_1810_11765_b200 import inputs as I
    a0 = I.gol_soup(W, H, p, seed)
    g = G.GameOfLife(a0, tiled=tiled)
    g.run(gens)
    assert np.array_equal(g.alive(), O.life_dense(a0, gens))
    assert g.heap.check_invariants() == 0


@pytest.mark.parametrize("tiled", ["prepare", "all"])
@pytest.mark.parametrize("P,W,H,gens", [(2, 64, 64, 60), (4, 130, 40, 50)])
def test_gol_tiled_row_shards_loopback_equal_dense(G, O, P, W, H, gens, tiled):
    from paper_1810_11765_b200 import inputs as I
    from paper_1810_11765_b200.gol import GameOfLifeLoopback
    a0 = I.gol_soup(W, H, 0.3, P + 30)
    lb = GameOfLifeLoopback(a0, P, tiled=tiled)
    lb.run(gens)
    assert np.array_equal(lb.alive(), O.life_dense(a0, gens))
    for s in lb.shards:
        assert s.heap.check_invariants() == 0


@pytest.mark.slow
def test_gol_tiled_16384_equals_block_list_and_dense(G, O):
    """configs[3] size, 3 generations: the tiled passes give exactly the
    block-list passes' alive map, and the oracle's dense Life on windows."""
    from paper_1810_11765_b200 import inputs as I
    W = H = 16384
    a0 = I.gol_soup(W, H, 0.25, 42)
    g = G.GameOfLife(a0, tiled=True)
    g.run(3)
    got = g.alive()
    assert g.heap.check_invariants() == 0
    del g
    torch.cuda.empty_cache()
    rng = np.random.default_rng(5)
    for _ in range(6):
        y, x = int(rng.integers(0, H - 300)), int(rng.integers(0, W - 300))
        want = O.life_dense(np.ascontiguousarray(a0[y:y + 262, x:x + 262]), 3)[3:259, 3:259]
        assert np.array_equal(got[y + 3:y + 259, x + 3:x + 259], want)
    g = G.GameOfLife(a0)
    g.run(3)
    assert np.array_equal(got, g.alive())
