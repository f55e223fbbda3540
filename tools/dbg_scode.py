import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import port
from paper_1710_03940_b200 import problems, _native as nat
p = problems.poisson3d(100)
A = nat.CsrArrays(p.matrix.nrows, p.matrix.ncols, p.matrix.row_ptr, p.matrix.col_idx, p.matrix.values)
h = nat.Hierarchy(A, nat.AmgOptions(0.08, 2 / 3, 0.8, 1, 25, 500))
nr, nc, ptr, col, val = h.matrix(0, nat.LEVEL_R)
rl = np.diff(ptr)
print("R", nr, nc, "mean", rl.mean(), "max", rl.max(), "maxgap", max(np.diff(col[ptr[i]:ptr[i+1]]).max() for i in range(0, nr, 97) if rl[i] > 1))
R = nat.CsrArrays(nr, nc, ptr, col, val)
x = np.random.default_rng(11).standard_normal(nc)
y = nat.spmv_device(R, x)
ref = port.spmv(port.Csr(nr, nc, ptr, col, val), x)
bad = np.nonzero(y != ref)[0]
print("mismatches", len(bad), "of", nr)
for i in bad[:10]:
    print(i, rl[i], y[i], ref[i])
