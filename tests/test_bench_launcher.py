"""bench.py's multi-rank launcher and the reference arm's JSON line (CPU; no GPU needed).

`bench.py --gpus N` without WORLD_SIZE re-executes itself under torch.distributed.run with N ranks
(127.0.0.1 rendezvous); the reference arm (the oracle, tier contract ④) runs on rank 0 only and prints
the same metric string and config as our arm, so the driver can form the ratio."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_spawn_command_shape():
    cmd = bench.spawn_cmd(4, ["--gpus", "4", "--steps", "3"], 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1] == "29555"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")


def test_reference_arm_spawns_ranks_and_matches_metric():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 alone prints
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["impl"] == "reference" and d["metric"] == base["metric"] == bench.METRIC
    assert d["n_gpus"] == 2 and d["unit"] == "solves/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == bench.WORKLOAD and d["config"]["global_batch"] == 578
    assert d["scaling"] == "strong"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
