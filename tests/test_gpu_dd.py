"""GPU parity of config 5's octant domain decomposition against oracle/dd.py.

Reduced sizes the oracle finishes in seconds (n = 16 per octant, cap degree 4, interface degree 4);
tolerances of R23: B blocks <= 1e-11, PKS fields after the steps <= 1e-9, dt <= 1e-12 relative,
point sets and piece assignment bit-exact.
"""
import numpy as np
import pytest
import torch

from oracle import dd as odd

pytestmark = pytest.mark.gpu

N, LC, LI = 16, 4, 4
BOX = (-0.1, 1.1)


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


@pytest.fixture(scope="module")
def api():
    from paper_1811_03557_b200 import api as A
    assert torch.cuda.is_available()
    return A


@pytest.fixture(scope="module")
def setup():
    return odd.setup(N, LC, LI)


def test_octant_sets_and_pieces(api, setup):
    o = setup.octants[0]
    for s in (0, 3, 7):
        g = api.Octant(N, *BOX, s, 1.0, LC, LI, 1e-3)
        for w in ["mplus", "gamma", "gamma_in", "gamma_ex", "band", "nplus"]:
            assert np.array_equal(g.copy_set(w), o.ps.list(w)), w
        bits = g.copy_assign()
        ob = (o.assign * np.array([1, 2, 4, 8])).sum(axis=1)
        assert np.array_equal(bits, ob)
        assert g.K == setup.K and g.n_rows == len(o.rows)


@pytest.mark.parametrize("s", [0, 5])
def test_bep_block(api, setup, s):
    dt = 1e-3
    g = api.Octant(N, *BOX, s, 1.0, LC, LI, dt)
    B = g.bep_block(want=True).cpu().numpy().T          # n_rows x K
    Bo, _ = odd.bep_block(setup, setup.octants[s], dt)
    assert rel(B, Bo) <= 1e-11, rel(B, Bo)


def test_bep_block_from_reference_octant(api, setup):
    # dpm_dd_bep_block_from: octant s's block from octant 0's by the column signs of the extensions
    # (B_s = B_0 diag(S_s)) against the oracle's block of octant s and the GPU's own K AP solves
    dt = 1e-3
    g0 = api.Octant(N, *BOX, 0, 1.0, LC, LI, dt)
    g0.bep_block()
    for s in (1, 5, 7):
        g = api.Octant(N, *BOX, s, 1.0, LC, LI, dt)
        Bf = g.bep_block_from(g0, want=True).cpu().numpy().T
        Bo, _ = odd.bep_block(setup, setup.octants[s], dt)
        assert rel(Bf, Bo) <= 1e-11, (s, rel(Bf, Bo))
        Bd = g.bep_block(want=True).cpu().numpy().T
        assert rel(Bf, Bd) <= 1e-13, (s, rel(Bf, Bd))
    g1 = api.Octant(N, *BOX, 1, 1.0, LC, LI, 2e-3)   # reference block at another dt: refused
    with pytest.raises(Exception):
        g1.bep_block_from(g0)


def test_dd_pks_parity(api):
    from paper_1811_03557_b200.dd import DDSolver
    steps, cap = 3, 1e-3
    o = odd.DDPKSOracle(N, LC, LI, cap, steps)
    state, ologs = o.run()
    octs = [api.Octant(N, *BOX, s, 1.0, LC, LI, cap) for s in range(8)]
    sol = DDSolver(octs, cap)
    sol.init((0.0, 0.0, 0.0), (1000.0, 100.0), (500.0, 50.0))
    r0 = o.initial_state()
    for (rho, c), (ro, co) in zip(sol.fields, r0):
        assert rel(rho.cpu().numpy(), ro) <= 1e-13
        assert rel(c.cpu().numpy(), co) <= 1e-13
    logs = [sol.step() for _ in range(steps)]
    for (rho, c), (ro, co) in zip(sol.fields, state):
        assert rel(rho.cpu().numpy(), ro) <= 1e-9, rel(rho.cpu().numpy(), ro)
        assert rel(c.cpu().numpy(), co) <= 1e-9, rel(c.cpu().numpy(), co)
    for lg, lo in zip(logs, ologs):
        assert abs(lg["dt"] - lo["dt"]) <= 1e-12 * lo["dt"]
        assert abs(lg["mass"] - lo["mass"]) <= 1e-9 * abs(lo["mass"])
    assert sol.builds == o.builds


def test_dd_pks_parity_per_octant_abi_path(api):
    # The path every rank takes with ONE octant (8 GPUs): DDSolver's non-batched branch, i.e. the
    # per-octant dpm_dd_local_begin / dpm_dd_local_finish calls (their own scratch and launches), with the
    # coefficient sums formed across the 8 octant contexts as the all-reduce would across ranks.
    from paper_1811_03557_b200.dd import DDSolver
    steps, cap = 3, 1e-3
    o = odd.DDPKSOracle(N, LC, LI, cap, steps)
    state, ologs = o.run()
    octs = [api.Octant(N, *BOX, s, 1.0, LC, LI, cap) for s in range(8)]
    sol = DDSolver(octs, cap)
    sol._batched = lambda: False
    sol.init((0.0, 0.0, 0.0), (1000.0, 100.0), (500.0, 50.0))
    logs = [sol.step() for _ in range(steps)]
    for (rho, c), (ro, co) in zip(sol.fields, state):
        assert rel(rho.cpu().numpy(), ro) <= 1e-9, rel(rho.cpu().numpy(), ro)
        assert rel(c.cpu().numpy(), co) <= 1e-9, rel(c.cpu().numpy(), co)
    for lg, lo in zip(logs, ologs):
        assert abs(lg["dt"] - lo["dt"]) <= 1e-12 * lo["dt"]
        assert abs(lg["mass"] - lo["mass"]) <= 1e-9 * abs(lo["mass"])


def test_dd_lsq_rhs_shared_equals_per_octant(api):
    # dpm_dd_lsq_rhs_shared (one pass over octant 0's Q, B_s = B_0 diag(S_s)) against the sum of the
    # per-octant operators M_s g_s on the same particular solutions
    from paper_1811_03557_b200.dd import DDSolver
    from dpm_inputs.rng import random_boxes
    dt = 1e-3
    octs = [api.Octant(N, *BOX, s, 1.0, LC, LI, dt) for s in range(8)]
    sol = DDSolver(octs, dt)
    sol.build(dt)
    wk = torch.from_numpy(random_boxes(3, 16, N)).cuda()
    y = octs[0].dd_lsq_rhs_shared(octs, wk)
    ref = sum(o.dd_lsq_rhs(wk[2 * i:2 * i + 2]) for i, o in enumerate(octs))
    torch.cuda.synchronize()
    assert rel(y.cpu().numpy(), ref.cpu().numpy()) <= 1e-11, rel(y.cpu().numpy(), ref.cpu().numpy())
    # a rank's shard at 4 GPUs / 2 GPUs: the reference octant is not octant 0
    for sub in ([3, 5], [2, 4, 6, 7]):
        so = [octs[s] for s in sub]
        wks = torch.cat([wk[2 * s:2 * s + 2] for s in sub])
        y = so[0].dd_lsq_rhs_shared(so, wks)
        ref = sum(o.dd_lsq_rhs(wks[2 * i:2 * i + 2]) for i, o in enumerate(so))
        torch.cuda.synchronize()
        assert rel(y.cpu().numpy(), ref.cpu().numpy()) <= 1e-11, (sub, rel(y.cpu().numpy(), ref.cpu().numpy()))


def test_dd_green_rhs_shared_equals_per_octant(api):
    # dpm_dd_green_rhs_shared (one basis evaluation per γ point, parity classes + Walsh-Hadamard) against
    # every octant's own extension + Green RHS, on all 8 octants and on a rank-sized subset
    from paper_1811_03557_b200.dd import DDSolver
    from dpm_inputs.rng import random_boxes
    dt = 1e-3
    octs = [api.Octant(N, *BOX, s, 1.0, LC, LI, dt) for s in range(8)]
    DDSolver(octs, dt).build(dt)
    fq = torch.from_numpy(random_boxes(5, 16, N)).cuda()
    Cg = torch.from_numpy(np.random.default_rng(6).uniform(-1, 1, size=(2, octs[0].K))).cuda()
    for sub in (list(range(8)), [6, 1, 3]):
        so = [octs[s] for s in sub]
        fqs = torch.cat([fq[2 * s:2 * s + 2] for s in sub])
        for clamp in (0, 1):
            wk = torch.zeros_like(fqs)
            so[0].dd_green_rhs_shared(so, Cg, clamp, fqs, wk)
            ref = torch.zeros_like(fqs)
            for i, o in enumerate(so):
                o.dd_green_rhs(Cg, clamp, fqs[2 * i:2 * i + 2], ref[2 * i:2 * i + 2])
            torch.cuda.synchronize()
            assert rel(wk.cpu().numpy(), ref.cpu().numpy()) <= 1e-12, (sub, clamp, rel(wk.cpu().numpy(), ref.cpu().numpy()))
    # in place (wk == fq) on flux-kernel output, which is zero off M+ (where the band lies)
    rho = [torch.from_numpy(np.abs(random_boxes(7 + s, 1, N)[0])).cuda() for s in range(8)]
    c = [torch.from_numpy(np.abs(random_boxes(17 + s, 1, N)[0])).cuda() for s in range(8)]
    fq2 = torch.zeros((16, N, N, N), dtype=torch.float64, device="cuda")
    for i, o in enumerate(octs):
        o.dd_rhs(rho[i], c[i], 1.0, fq2[2 * i:2 * i + 2])
    ref = torch.zeros_like(fq2)
    for i, o in enumerate(octs):
        o.dd_green_rhs(Cg, 1, fq2[2 * i:2 * i + 2], ref[2 * i:2 * i + 2])
    octs[0].dd_green_rhs_shared(octs, Cg, 1, fq2, fq2)
    torch.cuda.synchronize()
    assert rel(fq2.cpu().numpy(), ref.cpu().numpy()) <= 1e-12
