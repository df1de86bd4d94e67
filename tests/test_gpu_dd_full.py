"""Config 5 at its configured size (n = 128 per octant, cap degree 12, interface degree 12, K = 884)
against the oracle, through the exact 8-fold reflection symmetry of cfg5's origin-centred IC
(oracle/dd.py DDPKSOracleSymmetric: one octant's arithmetic, the stacked least squares reduced through
the thin QR of B_0; pinned against the full 8-octant oracle in tests/test_oracle_dd.py).

Checks (R23): octant 0's BEP block at the first dt, all 884 columns, <= 1e-11; two coupled PKS steps,
the second with a Step-4b rebuild (the dt cap halved after step 1 so that dt strictly decreases,
P:431), fields of all 8 octants <= 1e-9, dt <= 1e-12, total mass <= 1e-9.  The oracle needs ~1800 AP
solves at n = 128 (a few minutes on the host cores)."""
import numpy as np
import pytest
import torch

from dpm_inputs import get_config
from oracle import dd as odd

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


@pytest.fixture(scope="module")
def run():
    from paper_1811_03557_b200 import api
    from paper_1811_03557_b200.dd import DDSolver
    assert torch.cuda.is_available()
    cfg = get_config("cfg5")
    assert (cfg.n, cfg.lmax, cfg.deg_if) == (128, 12, 12)
    o = odd.DDPKSOracleSymmetric(cfg.n, cfg.lmax, cfg.deg_if, cfg.dt, 2, rho_ic=cfg.ic_rho, c_ic=cfg.ic_c,
                                 center=cfg.ic_center)
    octs = [api.Octant(cfg.n, cfg.lo, cfg.hi, s, 1.0, cfg.lmax, cfg.deg_if, cfg.dt) for s in range(8)]
    sol = DDSolver(octs, cfg.dt, chi=cfg.chi)
    sol.init(cfg.ic_center, cfg.ic_rho, cfg.ic_c)
    ost = o.initial_state()
    out = {"K": octs[0].K, "n_rows": octs[0].n_rows, "logs": [], "ologs": []}
    for k in range(2):
        if k == 1:                      # force Step 4b on step 2 on both sides
            o.dt_cap = sol.dt_cap = 0.5 * out["ologs"][0]["dt"]
        out["logs"].append(sol.step())
        ost, lg = o.step(ost)
        lg["mass"] = o.mass(ost)
        out["ologs"].append(lg)
        if k == 0:
            out["B_gpu"] = octs[0].bep_block(want=True).cpu().numpy().T     # n_rows x K at dt_1
            out["B_oracle"] = o.B0.copy()
    out["fields"] = [(r.cpu().numpy(), c.cpu().numpy()) for r, c in sol.fields]
    out["oracle_fields"] = ost
    out["builds"] = (sol.builds, o.builds)
    return out


def test_cfg5_bep_block_full_size(run):
    assert run["K"] == 884 and run["n_rows"] == 44145              # SURVEY probe P9: 44,145 rows
    assert run["B_gpu"].shape == run["B_oracle"].shape
    assert rel(run["B_gpu"], run["B_oracle"]) <= 1e-11, rel(run["B_gpu"], run["B_oracle"])


def test_cfg5_two_coupled_steps_with_rebuild(run):
    assert run["builds"] == (2, 2)
    for lg, lo in zip(run["logs"], run["ologs"]):
        assert lg["rebuilt"] == lo["rebuilt"]
        assert abs(lg["dt"] - lo["dt"]) <= 1e-12 * lo["dt"]
        assert abs(lg["mass"] - lo["mass"]) <= 1e-9 * abs(lo["mass"])
    assert abs(run["ologs"][0]["dt"] / 5.117385661696162e-07 - 1) < 1e-9      # SURVEY probe P12's dt_0
    ro, co = run["oracle_fields"]
    for rho, c in run["fields"]:                                    # every octant, canonical frame
        assert rel(rho, ro) <= 1e-9, rel(rho, ro)
        assert rel(c, co) <= 1e-9, rel(c, co)
