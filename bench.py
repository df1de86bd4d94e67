#!/usr/bin/env python
"""bench.py — headline benchmark of the B200-native DPM hot path.

Metric (BASELINE.json): "fp64 auxiliary solves/sec at N=128 (HBM-roofline fraction);
PKS time steps/sec".  The headline `value` is config 4: batched N=128 fp64 auxiliary
solves (I/dt - Δ_h)u = q, dt = 1e-5, 578 RHS of seeded U(-1,1) values on the spherical
shell band around r = 1 (R21), scattered into dense boxes; inputs resident in HBM.
One "step" = one dpm_aux_solve_batch call over this rank's shard of the 578 RHS
(sharded by RHS across ranks, no data-path collective; the 578-RHS workload is fixed as N grows, so
"scaling": "strong" — see DESIGN.md §8).  With --gpus N > 1 and no WORLD_SIZE in the environment,
bench.py re-executes itself under torch.distributed.run with N ranks.
PKS steps/s for configs 2 and 3 are reported in the "pks" object (rank 0, N=1 only).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from dpm_inputs import get_config  # noqa: E402
from dpm_inputs.rng import cfg4_band_values  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "fp64 auxiliary solves/sec at N=128 (HBM-roofline fraction); PKS time steps/sec"   # BASELINE.json
WORKLOAD = ("cfg4: N=128 box [-1.1,1.1]^3, dt=1e-5, 578 RHS U(-1,1) on the r=1 shell band (R21), dense boxes "
            "in/out")
FP64_PEAK_TFLOPS = 37.0      # measured DFMA / DMMA.8x8x4 peak on this pool's B200 (profiles/r01/microbench_*.log)


def load_peaks():
    try:
        return json.load(open(PEAKS_FILE)), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


_POLLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
arg = sys.argv[1]
h = pynvml.nvmlDeviceGetHandleByUUID(arg) if arg.startswith("GPU-") else pynvml.nvmlDeviceGetHandleByIndex(int(arg))
get = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
while True:
    print("%.6f,%d,%d,%d" % (time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx, int(get(h))), flush=True)
    time.sleep(0.005)
"""


class ClockSampler:
    """SM clocks and throttle reasons DURING the timed region (B200_PROFILING.md clocks line): an NVML
    poller subprocess (5 ms, wall-clock stamped; unaffected by the GIL) started before the warm-up;
    only the samples between mark_start() and mark_end() are summarised."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index = str(index)
        try:   # NVML does not see CUDA_VISIBLE_DEVICES: address the device by its UUID
            import torch
            uid = str(torch.cuda.get_device_properties(index).uuid)
            self.index = uid if uid.startswith("GPU-") else "GPU-" + uid
        except Exception:
            pass
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _POLLER, self.index], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 10
            while not self.lines and time.time() < deadline and self.proc.poll() is None:
                time.sleep(0.01)   # first sample in: the poller is running
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        time.sleep(0.02)   # let the samples of the last few ms arrive

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for ln in list(self.lines):
            try:
                ts, f, m, bits = ln.split(",")
                ts, f, m, bits = float(ts), float(f), float(m), int(bits)
            except ValueError:
                continue
            if self.t0 is not None and not (self.t0 <= ts <= (self.t1 or ts)):
                continue
            sm.append(f)
            mx = m
            for nm in self.NAMES:
                if bits & self.BITS[nm]:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml poller, 5 ms"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def oracle_sample_rate(cfg, nsolves, vals, band):
    """Oracle AP solves (direct-summation DST, numpy fp64) on host cores: solves/s."""
    from oracle import ap, dpm
    g_h = (cfg.hi - cfg.lo) / (cfg.n + 1)
    t0 = time.perf_counter()
    for b in range(nsolves):
        q = dpm.scatter(vals[b % len(vals)], band, cfg.n)
        ap.solve(q, g_h, cfg.dt)
    dt = time.perf_counter() - t0
    return nsolves / dt, dt


def oracle_baseline(cfg, vals, band, per_rep=20, reps=5):
    """cpu_baseline (tier contract): the oracle as it stands on the host cores, one warm-up
    solve, then the median of `reps` repetitions of `per_rep` solves of the cfg4 RHS (a bounded sample)."""
    oracle_sample_rate(cfg, 1, vals, band)
    runs = [oracle_sample_rate(cfg, per_rep, vals, band) for _ in range(reps)]
    rates = sorted(r for r, _ in runs)
    return statistics.median(rates), sum(t for _, t in runs), per_rep, reps


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def workload_config(B, nb, n, world, field):
    return {"workload": WORKLOAD, "global_batch": B, "local_batch": nb, "n": n, "parallelism": f"rhs-shard x{world}",
            "l2": "inputs larger than L2 (%.1f GB per rank per step)" % (nb * field * 8 / 1e9)}


def run_reference(args, world, rank):
    """--impl reference: the oracle, as it stands, on the host cores (rank 0 only; other ranks exit 0).
    Same metric, unit, config and higher_is_better as our arm; each step solves a bounded sample of 2 of
    the 578 cfg4 RHS (direct-summation DST)."""
    if rank != 0:
        return
    cfg = get_config("cfg4")
    from oracle import grid
    _, ps = grid.point_sets_for(cfg)
    band = ps.list("band")
    vals = cfg4_band_values(cfg.batch, len(band))
    per_step = 2
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=host_cores()):   # torchrun exports OMP_NUM_THREADS=1 to every rank
        for _ in range(args.warmup):
            oracle_sample_rate(cfg, 1, vals, band)
        times = []
        for _ in range(args.steps):
            _, t = oracle_sample_rate(cfg, per_step, vals, band)
            times.append(t)
    tot = sum(times)
    value = per_step * args.steps / tot
    n, B = cfg.n, cfg.batch
    per = -(-B // world)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(B, per, n, world, n ** 3),
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": host_cores(), "kind": "oracle",
                             "sample": f"{per_step} of the 578 cfg4 RHS per step (direct-summation DST, numpy)",
                             "model": cpu_model()},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_pks(api, torch, name, reps=20, hbm_peak=None):
    """the step loop repeated `reps` times from the same IC (median); setup
    (create + first BEP build) timed separately; hbm_frac against the ~96 N^3 B of a step (2 solves x 2
    fields x 16 N^3 + the stencil's reads and writes)."""
    cfg = get_config(name)
    ctx = api.DPM.from_config(cfg)
    n = cfg.n
    rho = torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
    c = torch.zeros_like(rho)
    t0 = time.perf_counter()
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
    ctx.pks_step(rho, c, 1, chi=cfg.chi, dt_cap=cfg.dt)      # builds the BEP at dt_0
    torch.cuda.synchronize()
    setup_ms = 1e3 * (time.perf_counter() - t0)
    per = []
    for _ in range(reps):
        ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        logs = ctx.pks_step(rho, c, cfg.steps, chi=cfg.chi, dt_cap=cfg.dt)
        torch.cuda.synchronize()
        per.append((time.perf_counter() - t0) / cfg.steps)
    ms = 1e3 * statistics.median(per)
    out = {"steps": cfg.steps, "reps": reps, "ms_per_step": ms, "steps_per_s": 1e3 / ms,
           "setup_ms_incl_bep_build": setup_ms, "rebuilds": sum(l["rebuilt"] for l in logs),
           "final_mass": logs[-1]["mass"], "rho_max": logs[-1]["rho_max"], "hbm_bytes_per_step": 96 * n ** 3}
    if hbm_peak:
        out["hbm_frac"] = 96 * n ** 3 * (1e3 / ms) / (hbm_peak * 1e9)
    return out


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def fps_reference_rate(cfg, vals, band, workers, nsolves=3):
    """A CPU fast-Poisson-solver reference analogous to the paper's FFTW3 + OpenMP, SURVEY §8(d):
    scipy.fft.dstn / idstn (type 1) with `workers` threads and the eigenvalue divide; solves/s.  Timing
    context only (not the oracle, not the product path)."""
    import scipy.fft as sf
    n, h = cfg.n, (cfg.hi - cfg.lo) / (cfg.n + 1)
    lam = (4.0 / h ** 2) * np.sin(np.arange(1, n + 1) * np.pi / (2 * (n + 1))) ** 2
    D = 1.0 / cfg.dt + lam[:, None, None] + lam[None, :, None] + lam[None, None, :]
    q = np.zeros(n ** 3)
    q[band] = vals[0]
    q = q.reshape(n, n, n)
    sf.idstn(sf.dstn(q, type=1, workers=workers) / D, type=1, workers=workers)   # warm-up
    t0 = time.perf_counter()
    for _ in range(nsolves):
        sf.idstn(sf.dstn(q, type=1, workers=workers) / D, type=1, workers=workers)
    return nsolves / (time.perf_counter() - t0)


def bench_cfg1(api, torch, reps=20):
    """cfg1 latency: the 51-RHS AP batch (50 basis potentials + 1 particular), the
    projection build (S2-S5) and the boundary LSQ (S8), N=16; median over reps, CUDA events."""
    from dpm_inputs.rng import cfg1_particular_values
    cfg = get_config("cfg1")
    ctx = api.DPM.from_config(cfg)
    n = cfg.n
    mp = ctx.copy_set("mplus")
    qp = np.zeros(n ** 3)
    qp[mp] = cfg1_particular_values(len(mp))
    E, _ = ctx.copy_extension()
    q = torch.cat([ctx.potential_rhs(torch.from_numpy(np.ascontiguousarray(E.T)).cuda()),
                   torch.from_numpy(qp.reshape(1, n, n, n)).cuda()])
    u = torch.empty_like(q)
    res = {}
    for name, fn in (("aux_solve_batch_51_us", lambda: ctx.aux_solve_batch(q, u)),
                     ("build_projection_us", lambda: ctx.build_projection(False)),
                     ("boundary_lsq_us", lambda: ctx.boundary_lsq(ctx.trace(u[50:51], "gamma_in")))):
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[name] = statistics.median(ts)
    return res


def bench_bep(api, torch, reps=3):
    """NEXT-1: the Step-4b rebuild at the cfg4 geometry (K = 578 BEP columns, N=128):
    dpm_bep_columns over all K (the octant path of bep_sym.cu: reflection-symmetric sets, parity-definite
    columns, DPM_BEP_SYM=0 for the full-grid path) and the whole dpm_build_projection (columns + CholeskyQR2
    factorisation, block-diagonal by parity class on the octant path); median of reps, CUDA events."""
    cfg = get_config("cfg4")
    ctx = api.DPM.from_config(cfg)
    K = ctx.K
    res = {"K": K, "path": "full grid" if os.environ.get("DPM_BEP_SYM") == "0" else
           "octant (reflection symmetry, 8 parity classes)",
           "fused": os.environ.get("DPM_BEP_FUSED") != "0"}
    for name, fn in (("columns_ms", lambda: ctx.bep_columns(0, K)),
                     ("rebuild_ms", lambda: ctx.build_projection(False))):
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name] = statistics.median(ts)
    res["columns_per_s"] = K / (res["columns_ms"] / 1e3)
    return res


def bench_bep_distributed(ctx, torch, dist, world, rank, reps=3):
    """C1 at N > 1: parallel.build_projection_distributed (columns sharded over ranks, NCCL all-gather of
    B, local CholeskyQR2) at the cfg4 geometry; median of reps of the max over ranks."""
    from paper_1811_03557_b200 import parallel
    parallel.build_projection_distributed(ctx, world, rank)
    ts = []
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        parallel.build_projection_distributed(ctx, world, rank)
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ts.append(float(t.item()))
    c0, c1 = parallel.shard_range(ctx.K, world, rank)
    return {"K": ctx.K, "ranks": world, "columns_per_rank": c1 - c0, "build_ms": statistics.median(ts),
            "collective": "all_gather of the |gamma_in| x K reduced BEP (%s)" % dist.get_backend()}


def bench_test_b(N=127, harmonics=150):
    """NEXT-4: the paper's Test B single domain, the
    Step-4b-every-step regime near blow-up: PKS steps until Δ||ρ||∞ >= 1000; blow-up time
    against the paper's t_min (Table 7), steps/s of the whole run including the rebuilds."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
    import test_b
    res, logs = test_b.run(N, harmonics)
    return res


def bench_rebuild_every_step(api, torch, name="cfg3", steps=20):
    """NEXT-1: the Step-4b regime forced on every step — each step
    runs at a new Δt (fixed-dt rule at Δt_i = Δt_0 (1 - 1e-3 i)), so the BEP is rebuilt every step
    (K = 2 (L+1)^2 AP solves + the CholeskyQR2 factorisation) before the step itself; steps/s of the
    whole loop, CUDA events."""
    cfg = get_config(name)
    ctx = api.DPM.from_config(cfg)
    n = cfg.n
    rho = torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
    c = torch.zeros_like(rho)
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
    dt0 = ctx.pks_step(rho, c, 1, chi=cfg.chi, dt_cap=cfg.dt)[0]["dt"]
    ctx.pks_step(rho, c, 2, chi=cfg.chi, dt_cap=dt0 * 0.999, dt_rule=1)   # warm-up (graph capture)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rebuilt = 0
    e0.record()
    for i in range(steps):
        rebuilt += ctx.pks_step(rho, c, 1, chi=cfg.chi, dt_cap=dt0 * (1.0 - 1e-3 * (i + 2)), dt_rule=1)[0]["rebuilt"]
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"config": name, "K": ctx.K, "n": n, "steps": steps, "rebuilds": rebuilt, "ms_per_step": ms,
            "steps_per_s": 1e3 / ms, "what": "BEP rebuilt on every step (Step 4b), then the step"}


def bench_test_a_dd():
    """NEXT-3: the paper's two-subdomain DD (Case 1) — the DD columns of Tables
    1-3 on the paper's N1/N2 meshes against the N = 516 SD reference, and Table 6's R_S on B200 (context)."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
    import test_a_dd
    return {"tables": test_a_dd.run_tables(), "rs": test_a_dd.run_rs(sizes=(127,))}


def bench_test_a():
    """NEXT-2: the paper's Test A convergence of the max density (Table 3)
    on the paper's meshes N = 36/68/132/260 against its N = 516 reference run, ρ̄0 as cell averages (R36):
    E_rel and rates next to the paper's."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
    import test_a
    test_a.IC_CELL = True
    res = test_a.run((36, 68, 132, 260, 516))
    einf = test_a.run_einf()
    return {"reference": res["reference"], "ic": res["ic"],
            "rows": [{k: r.get(k) for k in ("N", "E_rel", "paper_E_rel", "rate", "wall_s")} for r in res["rows"]],
            "reference_wall_s": res["reference_run"]["wall_s"],
            "einf_tables_1_2": {"reference": einf["reference"], "rows": einf["rows"]}}


def bench_dd(api, torch, world, rank, steps=None, reps=5):
    """cfg5: the 8-octant DD (R24) — octants sharded over the ranks (8/world each), the global
    least squares and dt through NCCL all-reduces (DDSolver).  The 50-step loop is repeated `reps`
    times from the same IC; steps/s excludes the BEP builds, which are timed separately
    (3 per run expected, SURVEY probe P12); medians over the repeats."""
    from paper_1811_03557_b200.dd import DDSolver
    cfg = get_config("cfg5")
    steps = steps or cfg.steps
    per = 8 // world
    mine = range(rank * per, (rank + 1) * per)
    dev = torch.cuda.current_device()
    octs = [api.Octant(cfg.n, cfg.lo, cfg.hi, s, 1.0, cfg.lmax, cfg.deg_if, cfg.dt, device=dev) for s in mine]
    sol = DDSolver(octs, cfg.dt, chi=cfg.chi)
    runs = []
    for _ in range(reps):
        sol.init(cfg.ic_center, cfg.ic_rho, cfg.ic_c)
        t_build, logs, b_start = 0.0, [], sol.builds
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            b0, ts = sol.builds, time.perf_counter()
            logs.append(sol.step())
            torch.cuda.synchronize()
            if sol.builds > b0:
                t_build += time.perf_counter() - ts
        tot = time.perf_counter() - t0
        nb = sol.builds - b_start
        runs.append({"total_s": tot, "builds": nb, "build_s": t_build,
                     "steps_per_s": (steps - nb) / max(tot - t_build, 1e-9), "logs": logs})
    med = lambda k: statistics.median(r[k] for r in runs)   # noqa: E731
    logs = runs[-1]["logs"]
    out = {"octants": 8, "octants_per_rank": per, "n": cfg.n, "K": octs[0].K, "rows_per_octant": octs[0].n_rows,
           "steps": steps, "reps": reps, "total_s": med("total_s"), "builds": runs[-1]["builds"],
           "build_s_incl_their_steps": med("build_s"), "steps_per_s_excl_builds": med("steps_per_s"),
           "steps_per_s_incl_builds": steps / med("total_s"),
           "builds_shared": "octant 0's block by K AP solves, the others by column signs (dpm_dd_bep_block_from)"
           if os.environ.get("DPM_DD_SHARED") != "0" and per > 1 else "every octant by K AP solves",
           "dt_first": logs[0]["dt"], "dt_last": logs[-1]["dt"], "t_end": logs[-1]["t"],
           "mass_after_step1": logs[0]["mass"], "mass_end": logs[-1]["mass"], "rho_max_end": logs[-1]["rho_max"],
           "note": "non-physical config (SURVEY §0 item 6: IC spike at the 8-octant corner); matches probe P12"}
    del sol, octs
    torch.cuda.empty_cache()
    return out


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_cmd(n, argv, port):
    """The torchrun command bench.py re-executes itself under for --gpus N > 1 without WORLD_SIZE."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def spawn_ranks(n):
    """One process per GPU over NCCL (rank 0 prints the JSON line); NCCL's init lines go to stderr so the
    ranks can be counted."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    r = subprocess.run(spawn_cmd(n, sys.argv[1:], free_port()), env=env)
    sys.exit(r.returncode)


def main():
    ap_ = argparse.ArgumentParser()
    ap_.add_argument("--gpus", type=int, default=1)
    ap_.add_argument("--steps", type=int, default=5)
    ap_.add_argument("--warmup", type=int, default=3)
    ap_.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap_.add_argument("--no-e2e", action="store_true")
    ap_.add_argument("--no-cpu", action="store_true")
    ap_.add_argument("--no-pks", action="store_true")
    ap_.add_argument("--no-dd", action="store_true")
    args = ap_.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    world, rank, local = dist_setup()
    if "WORLD_SIZE" in os.environ and world != args.gpus and rank == 0:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)\n")
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    # Functional check of the N > 1 path on a box with ONE GPU (tests/test_gpu_multirank.py): every rank on
    # cuda:0 (DPM_BENCH_ONE_GPU=1) and the collectives over gloo (DPM_BENCH_BACKEND=gloo; NCCL refuses two
    # ranks on one device).  The kernels of different ranks never wait on one another (host-side
    # collectives only); such a run measures nothing about scaling and says so in the line.
    backend = os.environ.get("DPM_BENCH_BACKEND", "nccl")
    one_gpu = os.environ.get("DPM_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if backend != "nccl":
            dist.init_process_group(backend)
        else:
            try:   # bind the NCCL communicator to this rank's GPU
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            except TypeError:
                dist.init_process_group("nccl")
    from paper_1811_03557_b200 import api
    from paper_1811_03557_b200._lib import lib as L

    cfg = get_config("cfg4")
    n, B = cfg.n, cfg.batch
    ctx = api.DPM.from_config(cfg, device=local)
    band = ctx.copy_set("band")
    per = -(-B // world)
    b0, b1 = rank * per, min(B, (rank + 1) * per)
    nb = max(0, b1 - b0)
    vals = cfg4_band_values(B, len(band))[b0:b1]
    field = n ** 3
    q = torch.zeros((nb, field), dtype=torch.float64, device="cuda")
    if nb:
        q[:, torch.from_numpy(band).cuda()] = torch.from_numpy(vals).cuda()
    q = q.view(nb, n, n, n)
    u = torch.empty_like(q)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            ctx.aux_solve_batch(q, u)
        barrier()
        peaks, peaks_kind = load_peaks()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = L.dpm_launch_count()
        barrier()
        clk.mark_start()
        ev0.record(stream)
        for _ in range(args.steps):
            ctx.aux_solve_batch(q, u)
        ev1.record(stream)
        barrier()
        clk.mark_end()
    launches = L.dpm_launch_count() - l0
    ms_local = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_per_step = ms_total / args.steps
    value = B / (ms_per_step / 1e3)                      # whole-job solves/s (all ranks)
    alg_bytes = 16 * n ** 3                              # dense fp64 box in + out per solve
    hbm_peak = peaks["hbm_gbs"]
    clocks = clk.summary()
    # fp64 work of the path as built: prime-factor DST-I transforms at 2 x 2732 flop per
    # line of 128 (2x3x43 factorisation) - two x passes over n^2 lines, and with the FACR(1) plane
    # pass two y transforms over the n^2/2 odd-z lines plus ~15 flop/point of recurrences (reduced
    # RHS, reduced z tridiagonal, even-z y tridiagonal); the full-transform plane kernel
    # (DPM_PLANE_FACR=0): four transforms + ~7 flop/point
    if os.environ.get("DPM_PLANE_FACR") == "0":
        flops_per_solve = 4 * n * n * 2 * 2732 + 7 * n ** 3
    else:
        flops_per_solve = 3 * n * n * 2 * 2732 + 15 * n ** 3

    # Per-kernel roofline of the dominant kernel: the same solves again with pass timing enabled
    # (CUDA events recorded by the library on this stream around every pass), right after the
    # timed region; algorithmic bytes per launch = 16 B x points of the launch (read + write once).
    ctx.set_pass_timing(True)
    for _ in range(max(1, min(args.steps, 2))):
        ctx.aux_solve_batch(q, u)
    torch.cuda.synchronize()
    pt = ctx.pass_times()
    ctx.set_pass_timing(False)
    kind = max(pt, key=lambda k: pt[k][0])
    k_ms, k_launch, k_pts = pt[kind]
    k_avg_s = k_ms / max(k_launch, 1) / 1e3
    k_bytes = 16.0 * k_pts / max(k_launch, 1)
    k_gbs = k_bytes / k_avg_s / 1e9 if k_avg_s > 0 else 0.0
    share = k_ms / max(sum(v[0] for v in pt.values()), 1e-30)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
    if not os.path.exists(tfile):
        tfile = os.path.join(ROOT, "profiles", "r01", "ncu_traffic.json")
    if os.path.exists(tfile):
        tr = json.load(open(tfile)).get(kind)
        if tr and tr.get("points_per_launch"):
            traffic = tr["dram_bytes_per_launch"] * (k_pts / max(k_launch, 1)) / tr["points_per_launch"]
    kernel_names = {"x": "dst128f_kernel<0> (prime-factor DST-I along x, DFMA)",
                    "y": ("plane128_kernel (fused y-DST / z tridiagonal / inverse y-DST per x-mode plane, 2-CTA "
                          "clusters)" if os.environ.get("DPM_PLANE_FACR") == "0" else
                          "plane128_facr_kernel (fused plane pass with one cyclic-reduction level along z: y-DST "
                          "of the 64 odd z, reduced z tridiagonal, inverse y-DST, y tridiagonal solves for the "
                          "even z; 2-CTA clusters)") if pt["z"][1] == 0
                         else "dst128f_kernel<1> (prime-factor DST-I along y, DFMA)",
                    "z": "ztri_warp_kernel<128> (exact tridiagonal solve along z)"}

    line = {"metric": METRIC,
            "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(B, nb, n, world, field),
            "roofline": {"bound": "hbm", "kernel": kernel_names.get(kind, kind), "achieved": k_gbs, "peak": hbm_peak,
                         "unit": "GB/s", "frac": k_gbs / hbm_peak, "traffic": traffic,
                         "peak_kind": peaks_kind + " (MEASURED_PEAKS.json hbm_gbs, burst copy)",
                         "alg_bytes_per_launch": k_bytes, "launch_ms": k_avg_s * 1e3, "share_of_step": share,
                         "passes": {k: {"ms": v[0], "launches": v[1], "points": v[2]} for k, v in pt.items()},
                         "path": {"what": "whole AP solve (x pass, fused plane pass, x pass) per dpm_aux_solve_batch",
                                  "achieved": alg_bytes * value / world / 1e9 if world else 0.0,
                                  "frac": alg_bytes * value / world / 1e9 / hbm_peak,
                                  "alg_bytes_per_solve": alg_bytes},
                         "fp64": {"achieved_tflops": flops_per_solve * value / world / 1e12,
                                  "peak_tflops": FP64_PEAK_TFLOPS,
                                  "frac": flops_per_solve * value / world / 1e12 / FP64_PEAK_TFLOPS,
                                  "flops_per_solve": flops_per_solve}},
            "gpu_launches": int(launches), "clocks": clocks}
    if world > 1 and (one_gpu or backend != "nccl"):
        line["functional_only"] = ("%d ranks, backend %s%s: a check of the multi-rank path, not a scaling number"
                                   % (world, backend, ", all on cuda:0" if one_gpu else ""))

    if not args.no_e2e and nb:
        # e2e through the C-ABI host-buffer call: pinned host q/u, H2D + solve + D2H inside the timed region
        qh = torch.empty((nb, n, n, n), dtype=torch.float64, pin_memory=True)
        qh.copy_(q)
        uh = torch.empty_like(qh, pin_memory=True)
        ctx.aux_solve_batch_host(qh, uh)
        barrier()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 2))
        for _ in range(e2e_steps):
            ctx.aux_solve_batch_host(qh, uh)
        barrier()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e_ms = float(el.item()) * 1e3 / e2e_steps
        line["e2e"] = {"value": B / (e2e_ms / 1e3), "unit": "solves/s", "h2d_bytes_per_step": nb * field * 8,
                       "d2h_bytes_per_step": nb * field * 8, "ms_per_step": e2e_ms,
                       "path": "dpm_aux_solve_batch_host (pinned host buffers)"}
        del qh, uh

    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import grid
        _, ps = grid.point_sets_for(cfg)
        band = ps.list("band")
        rate, secs, per_rep, reps = oracle_baseline(cfg, vals[:20], band)
        line["cpu_baseline"] = {"value": rate, "unit": "solves/s", "cores": host_cores(), "kind": "oracle",
                                "sample": "median of %d repetitions of %d of the 578 cfg4 RHS after 1 warm-up solve "
                                          "(direct-summation DST, numpy BLAS), %.1f s" % (reps, per_rep, secs),
                                "model": cpu_model()}
        try:   # the same oracle on one BLAS thread, and a scipy.fft fast-Poisson reference
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                r1, s1 = oracle_sample_rate(cfg, 1, vals[:1], band)
            line["cpu_baseline"]["one_core"] = {"value": r1, "sample": "1 RHS, %.1f s" % s1}
            line["cpu_baseline"]["fps_reference"] = {
                "what": "scipy.fft dstn/idstn type 1 + eigenvalue divide (the paper's FFTW3 + OpenMP analogue)",
                "value": fps_reference_rate(cfg, vals, band, host_cores()), "workers": host_cores(),
                "value_1_worker": fps_reference_rate(cfg, vals, band, 1), "unit": "solves/s"}
        except Exception as e:   # timing context only
            line["cpu_baseline"]["extra_error"] = repr(e)

    if rank == 0 and world == 1 and not args.no_pks:
        del q, u
        torch.cuda.empty_cache()
        line["pks"] = {"cfg2": bench_pks(api, torch, "cfg2", hbm_peak=hbm_peak),
                       "cfg3": bench_pks(api, torch, "cfg3", hbm_peak=hbm_peak)}
        line["cfg1"] = bench_cfg1(api, torch)
        line["bep_rebuild_cfg4"] = bench_bep(api, torch)
        line["pks_rebuild_every_step"] = bench_rebuild_every_step(api, torch)
        line["test_b"] = bench_test_b()
        line["test_a"] = bench_test_a()
        line["test_a_dd"] = bench_test_a_dd()

    if world > 1:
        # C1: one BEP build of the cfg4 geometry with its K = 578 columns sharded over the
        # ranks, one all-gather of B, redundant factorisation on every rank; CUDA events, max over ranks
        try:
            del q, u
        except NameError:
            pass
        torch.cuda.empty_cache()
        try:
            line["bep_build_distributed_cfg4"] = bench_bep_distributed(ctx, torch, dist, world, rank)
        except Exception as e:   # the headline above stands; the error is reported in its place
            line["bep_build_distributed_cfg4"] = {"error": repr(e)}

    if not args.no_dd and 8 % world == 0:
        try:
            del q, u
        except NameError:
            pass
        torch.cuda.empty_cache()
        try:
            dd = bench_dd(api, torch, world, rank)
        except Exception as e:
            if world == 1:
                raise
            dd = {"error": repr(e)}
        if rank == 0:
            line["dd"] = {"cfg5": dd}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
