"""The scaling-sweep harness (paper_1710_03940_b200.sweep) against the
reference CLI's contract (pkg/src/deflamg/cli.py:48-51, 216-289) and its
recorded acceptance numbers (c04, pkg/test_output.txt:348)."""
import pytest

from paper_1710_03940_b200 import SolverConfig
from paper_1710_03940_b200 import sweep


def test_csv_headers_are_the_references():
    assert sweep.BENCH_CSV_HEADER == "subdomains,threads,setup_s,factorize_E_s,solve_s,iters,converged"
    assert sweep.COMPARE_CSV_HEADER == (
        "subdomains,unknowns,deflated_iters,deflated_converged,local_iters,local_converged")
    assert sweep.csv_text("a,b", [(1, "x"), (2, "y")]) == "a,b\n1,x\n2,y\n"
    assert sweep._per_kind_path("out.csv", "linear", True) == "out-linear.csv"
    assert sweep._per_kind_path("out.csv", "linear", False) == "out.csv"


def test_argument_errors_exit_2(capsys):
    assert sweep.main(["bench", "--poisson", "8", "--subdomains", "1,x"]) == 2
    assert "expected integers" in capsys.readouterr().err
    assert sweep.main(["bench", "--poisson", "8", "--subdomains", "0"]) == 2
    assert sweep.main(["bench", "--poisson", "8", "--subdomains", "1", "--deflation", "quadratic"]) == 2
    assert sweep.main(["compare-deflation", "--poisson", "8", "--subdomains", "2", "--config", "/no/such"]) == 2


@pytest.mark.gpu
def test_c04_weak_sweep_compare_deflation():
    """c04 (test_acceptance.py:191-245): weak scaling at 12^3 per subdomain,
    m = 1/8/27, BiCGStab(2) + SPAI-0 + linear deflation, tol 1e-6: the
    reference records deflated [3, 6, 6] and plain block-AMG [3, 7, 10]."""
    cfg = SolverConfig({"solver": {"type": "bicgstab2", "tol": 1e-6}, "precond": {"relax": {"type": "spai0"}},
                        "deflation": {"kind": "linear"}})
    rows = sweep.compare_deflation(12, [1, 8, 27], cfg)
    assert [r[0] for r in rows] == [1, 8, 27]
    assert [r[1] for r in rows] == [12 ** 3, 8 * 12 ** 3, 27 * 12 ** 3]
    for r, d, p in zip(rows, [3, 6, 6], [3, 7, 10]):
        assert r[3] == "true" and r[5] == "true"
        assert abs(r[2] - d) <= 1 and abs(r[4] - p) <= 1, r


@pytest.mark.gpu
def test_bench_sweep_rows(tmp_path):
    out = tmp_path / "b.csv"
    assert sweep.main(["bench", "--mode", "weak", "--poisson", "10", "--subdomains", "1,2",
                       "--deflation", "constant,linear", "--csv", str(out)]) == 0
    for kind in ("constant", "linear"):
        lines = (tmp_path / f"b-{kind}.csv").read_text().splitlines()
        assert lines[0] == sweep.BENCH_CSV_HEADER and len(lines) == 3
        cells = lines[2].split(",")
        assert cells[0] == "2" and cells[-1] == "true" and int(cells[5]) > 0
