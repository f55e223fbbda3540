"""Projector accuracy on the rhs, GPU vs the CPU oracle: b' = P b, its
Z-orthogonality (Z'b' evaluated in long double), and the coarse lift of b.

    python tools/diag_proj.py KIND EDGE M [relax]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import port  # noqa: E402
from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver  # noqa: E402

kind, edge, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
relax = sys.argv[4] if len(sys.argv) > 4 else ("damped_jacobi" if kind == "jump" else "spai0")
cfgd = {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": relax}}, "deflation": {"kind": "linear"}}
p = problems.make_problem(edge, problems.boxes_for(m), kind)
port.set_threads(os.cpu_count() or 1)
s = DeflatedSolver(p.matrix, p.partition, config=SolverConfig(cfgd), coords=p.coords)
o = port.DeflatedSolverOracle(p.matrix, p.partition, config=SolverConfig(cfgd), coords=p.coords)
Zt = o.basis.Zt


def zt_ld(v):
    """Z' v in long double (80-bit) from the oracle's Zt CSR."""
    out = np.zeros(Zt.nrows, dtype=np.longdouble)
    for j in range(Zt.nrows):
        a, b = Zt.row_ptr[j], Zt.row_ptr[j + 1]
        out[j] = np.sum(Zt.values[a:b].astype(np.longdouble) * v[Zt.col_idx[a:b]].astype(np.longdouble))
    return out


b = p.rhs
res = {}
bp, bpo = s.project(b), o.project(b)
res["bprime_rel_diff"] = float(np.linalg.norm(bp - bpo) / np.linalg.norm(bpo))
res["Zt_bprime_gpu"] = float(np.linalg.norm(zt_ld(bp)))
res["Zt_bprime_oracle"] = float(np.linalg.norm(zt_ld(bpo)))
res["Zt_b"] = float(np.linalg.norm(zt_ld(b)))
t_ld = zt_ld(b)
t_o = port.spmv(Zt, b)
res["t_oracle_err"] = float(np.linalg.norm(t_o - t_ld.astype(np.float64)))
res["t_abs"] = [float(v) for v in t_ld[:8]]
lf, lfo = s.coarse_lift(b), o.coarse_lift(b)
res["lift_rel_diff"] = float(np.linalg.norm(lf - lfo) / np.linalg.norm(lfo))
E = o.basis.E
res["E_rel_diff"] = float(np.linalg.norm(s.basis.E - E) / np.linalg.norm(E))
res["E_max_abs_diff"] = float(np.abs(s.basis.E - E).max())
res["cond_E"] = float(np.linalg.cond(E))
# exact-ish coarse solve in long double from the long-double t and E
tl = t_ld.astype(np.float64)
y_lu = o.basis.lu.solve(tl)
res["t2_gpuE_vs_oracleE"] = float(np.linalg.norm(np.linalg.solve(s.basis.E, tl) - y_lu) / np.linalg.norm(y_lu))
print(json.dumps(res), flush=True)
