"""cProfile of DeflatedSolver construction (host setup + upload + layout
conversion) at 150^3 on one B200."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402,F401  (imported by the bench before the setup too)

from paper_1710_03940_b200 import DeflatedSolver, SolverConfig, problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 150
p = problems.poisson3d(n)
cfg = SolverConfig({"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
                    "deflation": {"kind": "linear"}})
DeflatedSolver(problems.poisson3d(12).matrix, problems.poisson3d(12).partition, config=cfg,
               coords=problems.poisson3d(12).coords, device=0)
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
s = DeflatedSolver(p.matrix, p.partition, config=cfg, coords=p.coords, device=0)
pr.disable()
print(f"construction {time.perf_counter() - t:.3f} s, setup_seconds {s.setup_seconds:.3f}")
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
