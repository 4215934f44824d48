"""Write tests/golden/nbody65536_10steps.npz: the oracle's state after 10
steps of BASELINE configs[2] (65,536 bodies, seed 7, inputs.NBODY_PARAMS,
merges on).  Calls only oracle/ (and the seeded input generator); the GPU
path never writes or reads anything here except in the comparison test
(tests/test_gpu_apps.py::test_nbody_65536_ten_steps_baseline_config).
Takes ~10 min on one core: python scripts/make_nbody_golden.py"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O                      # noqa: E402
from paper_1810_11765_b200 import inputs as I       # noqa: E402

N, SEED, STEPS = 65536, 7, 10
O.build()
st = I.nbody_init(N, seed=SEED)
t0 = time.time()
w = O.nbody_run(st, merges=True, steps=STEPS, **I.NBODY_PARAMS)
out = ROOT / "tests" / "golden" / "nbody65536_10steps.npz"
np.savez_compressed(out, x=w["x"], y=w["y"], vx=w["vx"], vy=w["vy"], m=w["m"], alive=w["alive"],
                    meta=np.array([N, SEED, STEPS]),
                    params=np.array([I.NBODY_PARAMS[k] for k in ("G", "dt", "eps", "R")]))
print(f"wrote {out} ({out.stat().st_size} B) in {time.time() - t0:.0f} s; survivors {int(w['alive'].sum())}")
