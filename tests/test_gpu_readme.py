"""The README's usage example runs as written (GPU)."""
import os

import pytest

pytestmark = pytest.mark.gpu


def test_readme_example_runs():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "README.md")).read()
    a = text.index("```python") + len("```python")
    code = text[a:text.index("```", a)]
    ns = {}
    exec(compile(code, "README.md", "exec"), ns)
    assert ns["u"].shape == (4, 128, 128, 128)
    assert ns["coef"].shape == (4, ns["ctx"].K)
    assert len(ns["logs"]) == 10 and all(l["mass"] > 0 for l in ns["logs"])
    assert ns["diag"]["free_energy"] < 0 or ns["diag"]["free_energy"] > 0   # finite
    assert len(ns["ta_logs"]) == 100 and abs(ns["ta_logs"][-1]["t"] - 1e-6) < 1e-18
    assert abs(ns["ta_logs"][-1]["rho_max_mplus"] - 1126.89) < 0.05   # ||ρ̄||∞ at T on N = 68, cell-average IC
    assert len(ns["dd_logs"]) == 10 and abs(ns["dd_logs"][-1]["t"] - 1e-7) < 1e-20
    assert ns["dd_logs"][-1]["rho_max_mplus"] > 900                   # the centre of Ω1 carries max ρ
