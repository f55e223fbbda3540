"""Host vs device setup products at 150^3 (one B200): hierarchy build time."""
import sys
import time

sys.path.insert(0, ".")
from paper_1710_03940_b200 import _native as nat, problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 150
p = problems.poisson3d(n)
A = nat.CsrArrays(p.matrix.nrows, p.matrix.ncols, p.matrix.row_ptr, p.matrix.col_idx, p.matrix.values)
opts = nat.AmgOptions(0.08, 2 / 3, 0.8, nat.DFL_RELAX["spai0"], 25, 500)
w = problems.poisson3d(10).matrix
nat.Hierarchy(nat.CsrArrays(w.nrows, w.ncols, w.row_ptr, w.col_idx, w.values), opts, device=0)  # CUDA warm-up
for dev in (0, None, 0, None, 0):
    t = time.perf_counter()
    h = nat.Hierarchy(A, opts, device=dev)
    print(f"{n}^3 hierarchy ({'device' if dev is not None else 'host'} products): "
          f"{time.perf_counter() - t:.3f} s, levels {h.level_sizes}", flush=True)
