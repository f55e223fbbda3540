"""BASELINE configs at full size, on one B200, against the REFERENCE's own
results at the same subdomain counts (tests/golden/configs, written by
tests/golden/make_golden_configs.py running deflamg itself).

The m subdomains of a config run as S = m subdomains on one GPU (their AMG
hierarchies merged block-diagonally, the deflation space K = m*k exactly as
the reference builds it, deflation.py:83-163), so the iteration counts that
the weak/strong-scaling claims rest on (config #2: 23/63/69/101 at
m = 1/2/4/8; #3: 30/30 at m=1 ... 99/92 at m=8; #4: 67/65; #5: 22/16) are
checked on the device.

Parity rule (BASELINE.md note ‡): same stopping rule (converged on the
recurrence residual), iterations within ±1, true relative residual
<= max(tol, 2 x the reference's), and rel-L2(x - x_ref) <= 1e-6 on the
reference's x (sampled at 16384 evenly spaced unknowns; |x| and sum(x) are
exact).  Config #5 at m=1 is the one case where the reference's own x is
inaccurate (its BiCGStab(2) recurrence stagnates: true residual 2.5e-7 for a
1e-8 target), so there both solutions are compared with a 1e-12 solve and
ours must be at least as close.
"""
import glob
import json
import os

import numpy as np
import pytest

from paper_1710_03940_b200 import _native as nat
from paper_1710_03940_b200 import problems
from paper_1710_03940_b200.config import SolverConfig
from paper_1710_03940_b200.deflation import DeflatedSolver

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "configs")
CASES = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(HERE, "*.json")))


def _load(case):
    with open(os.path.join(HERE, case + ".json")) as fh:
        meta = json.load(fh)
    z = np.load(os.path.join(HERE, case + ".npz"))
    return meta, z["idx"], z["x"]


_ROWS = {}


def _rows(kind, shape, boxes):
    key = (kind, tuple(shape), tuple(boxes))
    if key not in _ROWS:
        _ROWS.clear()  # one problem at a time (a 300^3 problem is ~0.7 GB of host CSR)
        o = problems.BoxOrdering(tuple(shape), tuple(boxes))
        ptr, col, val, coords = nat.gen_rows(0, o.shape, o.boxes, kind, 0, o.n)  # on the GPU, bit-identical
        _ROWS[key] = (o, (ptr, col, val), coords)
    return _ROWS[key]


def _solve(meta, tol=None):
    o, rows, coords = _rows(meta["kind"], meta["shape"], meta["boxes"])
    cfgd = json.loads(json.dumps(meta["config"]))
    if tol is not None:
        cfgd["solver"]["tol"] = tol
        cfgd["solver"]["maxiter"] = 5000
    s = DeflatedSolver.from_rows(rows, o.n, o.partition(), config=SolverConfig(cfgd), coords_local=coords, device=0)
    h = 1.0 / (o.shape[0] + 1)
    x, rep = s.solve(np.full(o.n, h * h))
    return s, x, rep


@pytest.mark.parametrize("case", CASES)
def test_config_matches_reference(case):
    meta, idx, xs = _load(case)
    s, x, rep = _solve(meta)
    assert s.partition.m == meta["m"]
    assert s.basis.n_coarse == meta["K"]
    assert s.hierarchies[0].level_sizes == meta["levels"]
    assert meta["converged"] and rep["converged"]
    tol = meta["config"]["solver"]["tol"]
    assert rep["relative_residual"] <= max(tol, 2 * meta["relative_residual"]), rep["relative_residual"]
    if case == "c5_m1":
        # BASELINE.md ‡: the reference's recurrence residual drifts away from
        # its true residual (2.5e-7 for a 1e-8 target) and its group count
        # depends on the BLAS (22 single-threaded, 28 on the GPU host's
        # threaded BLAS), so the count is not a parity target here: ours
        # must stop no later, meet tol on the TRUE residual, and be at least
        # as close to a 1e-12 solution as the reference's x
        assert rep["iterations"] <= meta["iterations"] + 1
        assert rep["relative_residual"] <= tol
        # the oracle (the reference's algorithm, pinned bitwise to it) with only
        # its Z' r sums taken pairwise instead of sequentially over the 7M rows
        # converges in 9 groups to 9.0e-9 (tools/diag_zt_accuracy.py, committed
        # in tests/golden/c5_m1_zt_accuracy.json): the device matches that
        with open(os.path.join(os.path.dirname(HERE), "c5_m1_zt_accuracy.json")) as fh:
            acc = json.load(fh)
        assert acc["reference_sums"]["iters"] == meta["iterations"]
        assert abs(rep["iterations"] - acc["pairwise_zt"]["iters"]) <= 1, (rep["iterations"], acc["pairwise_zt"])
        _, xt, rt = _solve(meta, tol=1e-12)
        assert rt["converged"] and rt["relative_residual"] <= 1e-10
        e_gpu = np.linalg.norm(x[idx] - xt[idx])
        e_ref = np.linalg.norm(xs - xt[idx])
        assert e_gpu <= e_ref, (e_gpu, e_ref)
        assert np.linalg.norm(x - xt) / np.linalg.norm(xt) <= 1e-6
        return
    assert abs(rep["iterations"] - meta["iterations"]) <= 1, (rep["iterations"], meta["iterations"])
    rel = np.linalg.norm(x[idx] - xs) / np.linalg.norm(xs)
    assert rel <= 1e-6, rel
    assert abs(np.linalg.norm(x) - meta["x_norm"]) <= 1e-6 * meta["x_norm"]
    assert abs(x.sum() - meta["x_sum"]) <= 1e-6 * abs(meta["x_sum"])
