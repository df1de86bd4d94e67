"""The N > 1 paths on hardware with one GPU: W processes on cuda:0, host-side collectives over gloo.

NCCL cannot place two ranks on one device and the GPU box has one GPU, so these runs exercise everything
of the multi-rank path but NCCL itself: the distributed BEP build (C1) on CUDA tensors, the DD with the
octants sharded over processes (W = 8: the per-octant dpm_dd_local_begin/finish path every rank of an
8-GPU run takes) and bench.py's own --gpus N line.  They are functional checks, not scaling numbers."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


def _json_line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-3000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("world", [2, 8])
def test_multirank_bep_and_dd_match_single_rank(world):
    sys.path.insert(0, ROOT)
    import bench
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(bench.free_port()),
           os.path.join(ROOT, "tests", "helpers", "multirank_gpu_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    assert d["world"] == world
    assert d["bep_B_equal"] and d["bep_coef_rel"] <= 1e-12, d
    assert d["dd_path"] == ("batched" if world == 2 else "per-octant local_begin/finish")
    assert d["dd_builds"] == d["dd_builds_single"] >= 2
    assert d["dd_dt_rel"] <= 1e-12 and d["dd_mass_rel"] <= 1e-9 and d["dd_field_rel"] <= 1e-9, d   # R23


def test_bench_gpus_2_line_on_one_gpu():
    # bench.py --gpus 2 spawns its own ranks (no WORLD_SIZE): cfg4 shards, the distributed BEP build and the
    # cfg5 DD with 4 octants per rank; the line must carry them and reproduce the single-rank cfg5 trajectory
    env = _env()
    env.update(DPM_BENCH_BACKEND="gloo", DPM_BENCH_ONE_GPU="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3",
                        "--no-e2e"], capture_output=True, text=True, timeout=1200, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == base["metric"] and d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 578 and d["config"]["local_batch"] == 289
    assert "functional_only" in d and d["value"] > 0 and d["gpu_launches"] > 0
    b = d["bep_build_distributed_cfg4"]
    assert b["K"] == 578 and b["ranks"] == 2 and b["columns_per_rank"] == 289 and b["build_ms"] > 0
    dd = d["dd"]["cfg5"]
    assert dd["octants_per_rank"] == 4 and dd["K"] == 884 and dd["builds"] == 3
    # SURVEY probe P12 / the single-rank run: dt 5.1174e-7 -> 8.4348e-8, t_end 4.645e-6
    assert abs(dd["dt_first"] / 5.117385661696e-07 - 1) <= 1e-9
    assert abs(dd["dt_last"] / 8.434757742e-08 - 1) <= 1e-6
    assert abs(dd["t_end"] / 4.6449601e-06 - 1) <= 1e-6
