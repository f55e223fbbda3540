"""SolverConfig: the reference's key tree, defaults and validation
(pkg/src/deflamg/config.py; pkg/tests/test_config.py)."""
import json

import pytest

from paper_1710_03940_b200.config import DEFAULTS, SolverConfig
from paper_1710_03940_b200.errors import ConfigError


def test_defaults():
    c = SolverConfig()
    assert c.get("solver.type") == "bicgstab2" and c.get("solver.tol") == 1e-6
    assert c.get("precond.relax.type") == "damped_jacobi" and c.get("precond.relax.damping") == 0.8
    assert c.get("precond.coarsening.eps_strong") == 0.08 and c.get("precond.coarse_enough") == 500
    assert c.get("deflation.kind") == "constant" and c.get("deflation.inexact") is False


def test_merge_types_and_unknown_keys():
    c = SolverConfig({"solver": {"tol": 1, "maxiter": 20.0}})
    assert c.get("solver.tol") == 1.0 and isinstance(c.get("solver.maxiter"), int)
    for bad in ({"solver": {"tol": "x"}}, {"solver": {"maxiter": 2.5}}, {"nope": 1}, {"solver": 3},
                {"deflation": {"inexact": 1}}):
        with pytest.raises(ConfigError):
            SolverConfig(bad)
    with pytest.raises(ConfigError) as e:
        SolverConfig({"precond": {"relax": {"typo": 1}}})
    assert "precond.relax.typo" in str(e.value)


def test_set_get_json_roundtrip():
    c = SolverConfig().set("precond.relax.type", "spai0")
    assert SolverConfig.from_json(c.to_json()) == c
    with pytest.raises(ConfigError):
        c.set("precond.relax", 1)
    with pytest.raises(ConfigError):
        SolverConfig.from_json("[1]")
    assert json.loads(SolverConfig().to_json())["deflation"] == DEFAULTS["deflation"]


def test_matches_reference_defaults_if_available():
    ref = pytest.importorskip("deflamg.config")
    assert ref.DEFAULTS == DEFAULTS
