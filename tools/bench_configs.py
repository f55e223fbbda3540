"""Every BASELINE.json config on one B200 (the bench line covers configs[1]).

For each config: host setup time, device solve time (CUDA events, b resident),
iterations and true relative residual next to the reference's own numbers
measured in the build container.  One JSON object per line.

    python tools/bench_configs.py [--only 1,3c,3l,4,5] [--steps 5]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402  (device buffers for the b-resident timing)

from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver, solve_device  # noqa: E402

CG = {"type": "cg", "tol": 1e-8, "maxiter": 1000}
BICG = {"type": "bicgstab2", "tol": 1e-8, "maxiter": 1000}
CONFIGS = {
    # name: (kind, shape, m, config, reference iterations, reference relres, reference solve s)
    "1": ("poisson", 32, 4, {"solver": CG, "precond": {"relax": {"type": "spai0"}}, "deflation": {"kind": "constant"}},
          32, 5.19e-9, 0.083),
    "2": ("poisson", 150, 1, {"solver": CG, "precond": {"relax": {"type": "spai0"}}, "deflation": {"kind": "linear"}},
          23, 8.23e-9, 15.10),
    "3c": ("poisson", 256, 1, {"solver": CG, "precond": {"relax": {"type": "spai0"}},
                               "deflation": {"kind": "constant"}}, 30, 8.49e-9, 106.47),
    "3l": ("poisson", 256, 1, {"solver": CG, "precond": {"relax": {"type": "spai0"}},
                               "deflation": {"kind": "linear"}}, 30, 6.74e-9, 111.65),
    "4": ("jump", 200, 1, {"solver": CG, "precond": {"relax": {"type": "damped_jacobi"}},
                           "deflation": {"kind": "linear"}}, 67, 1.07e-8, 113.91),
    "5": ("convdiff", 192, 1, {"solver": BICG, "precond": {"relax": {"type": "spai0"}},
                               "deflation": {"kind": "linear"}}, 22, 2.51e-7, 130.53),
}


def run(name, steps):
    kind, shape, m, cfgd, ref_it, ref_rr, ref_s = CONFIGS[name]
    ordering = problems.BoxOrdering(shape, problems.boxes_for(m))
    n = ordering.n
    t0 = time.perf_counter()
    from paper_1710_03940_b200 import _native as nat

    ptr, col, val, coords = nat.gen_rows(0, ordering.shape, ordering.boxes, kind, 0, n)  # on the GPU
    rows = (ptr, col, val)
    gen = time.perf_counter() - t0
    s = DeflatedSolver.from_rows(rows, n, ordering.partition(), config=SolverConfig(cfgd), coords_local=coords)
    h = 1.0 / (ordering.shape[0] + 1)
    b = torch.full((n,), h * h, dtype=torch.float64, device="cuda")
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        rep = solve_device(s, b.data_ptr(), x.data_ptr())
    times = []
    for _ in range(steps):
        rep = solve_device(s, b.data_ptr(), x.data_ptr())
        times.append(rep.solve_seconds)
    solve = statistics.median(times)
    return {
        "config": name, "kind": kind, "shape": shape, "subdomains": m, "solver": cfgd["solver"]["type"],
        "deflation": cfgd["deflation"]["kind"], "relax": cfgd["precond"]["relax"]["type"], "unknowns": n,
        "iterations": rep.iterations, "ref_iterations": ref_it, "converged": bool(rep.converged),
        "relative_residual": rep.relative_residual, "ref_relative_residual": ref_rr,
        "solve_ms": solve * 1e3, "ms_per_iteration": solve * 1e3 / max(1, rep.iterations),
        "ref_solve_s_cpu_build_container": ref_s, "speedup_vs_ref": ref_s / solve,
        "host_setup_s": s.setup_seconds, "generate_s": gen, "device_gb": s.device_bytes / 1e9,
        "level_sizes": s.hierarchies[0].level_sizes,
    }


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=",".join(CONFIGS))
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    for name in a.only.split(","):
        print(json.dumps(run(name, a.steps)), flush=True)
