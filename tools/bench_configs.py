"""Every BASELINE.json config at the reference's subdomain counts on one B200
(the bench line covers configs[1] at m = N).

For each case of tests/golden/configs (reference fingerprints written by
tests/golden/make_golden_configs.py): device setup time, device solve time
(CUDA events, b resident), iterations and true relative residual next to the
reference's own numbers, and rel-L2 of x against the reference's sampled x.
One JSON object per line.

    python tools/bench_configs.py [--only c2_m8,c4_m8] [--steps 5]
"""
import argparse
import glob
import json
import os
import statistics
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402  (device buffers for the b-resident timing)

from paper_1710_03940_b200 import _native as nat  # noqa: E402
from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver, solve_device  # noqa: E402

GOLD = os.path.join(REPO, "tests", "golden", "configs")


def run(case, steps):
    with open(os.path.join(GOLD, case + ".json")) as fh:
        meta = json.load(fh)
    z = np.load(os.path.join(GOLD, case + ".npz"))
    o = problems.BoxOrdering(tuple(meta["shape"]), tuple(meta["boxes"]))
    n = o.n
    t0 = time.perf_counter()
    ptr, col, val, coords = nat.gen_rows(0, o.shape, o.boxes, meta["kind"], 0, n)  # on the GPU
    gen = time.perf_counter() - t0
    s = DeflatedSolver.from_rows((ptr, col, val), n, o.partition(), config=SolverConfig(meta["config"]),
                                 coords_local=coords, device=0)
    h = 1.0 / (o.shape[0] + 1)
    x, rep = s.solve(np.full(n, h * h))
    b = torch.full((n,), h * h, dtype=torch.float64, device="cuda")
    xd = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        solve_device(s, b.data_ptr(), xd.data_ptr())
    times = [solve_device(s, b.data_ptr(), xd.data_ptr()).solve_seconds for _ in range(steps)]
    solve = statistics.median(times)
    idx, xs = z["idx"], z["x"]
    return {
        "case": case, "kind": meta["kind"], "shape": meta["shape"], "subdomains": meta["m"],
        "solver": meta["config"]["solver"]["type"], "deflation": meta["config"]["deflation"]["kind"],
        "relax": meta["config"]["precond"]["relax"]["type"], "unknowns": n, "K": s.basis.n_coarse,
        "iterations": rep["iterations"], "ref_iterations": meta["iterations"], "converged": rep["converged"],
        "relative_residual": rep["relative_residual"], "ref_relative_residual": meta["relative_residual"],
        "x_rel_l2_vs_ref_sampled": float(np.linalg.norm(x[idx] - xs) / np.linalg.norm(xs)),
        "solve_ms": solve * 1e3, "ms_per_iteration": solve * 1e3 / max(1, rep["iterations"]),
        "ref_solve_s": meta["solve_seconds"], "speedup_vs_ref": meta["solve_seconds"] / solve,
        "setup_s": s.setup_seconds, "ref_setup_s": meta["setup_seconds"], "generate_s": gen,
        "device_gb": s.device_bytes / 1e9, "level_sizes": s.hierarchies[0].level_sizes,
        "ref_note": "reference solve/setup seconds: deflamg in the build container, 1 core, single-threaded BLAS",
    }


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    cases = a.only.split(",") if a.only else sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLD, "*.json")))
    for c in cases:
        print(json.dumps(run(c, a.steps)), flush=True)
