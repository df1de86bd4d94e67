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
