"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: RHS sharding and the
distributed BEP build (column blocks + all-gather), with the ORACLE supplying the columns."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_03557_b200.parallel import shard_range, distributed_bep


def test_shard_ranges_cover_exactly():
    for total in (0, 1, 7, 578, 884):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                a, b = shard_range(total, world, r)
                assert 0 <= a <= b <= total
                seen.extend(range(a, b))
            assert seen == list(range(total))
    assert [shard_range(578, 8, r) for r in (0, 7)] == [(0, 73), (511, 578)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dpm_inputs import get_config
    from oracle import dpm, grid
    cfg = get_config("cfg1")
    g, ps = grid.point_sets_for(cfg)
    E, *_ = dpm.extension_matrix(g, ps, cfg.kind, cfg.center, cfg.semi, cfg.lmax, cfg.basis)

    def columns(c0, c1):
        _, B, _ = dpm.projection_and_bep(E[:, c0:c1], g, ps, cfg.dt)
        return torch.from_numpy(np.ascontiguousarray(B.T))

    B = distributed_bep(columns, E.shape[1], world, rank)
    q.put((rank, B.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_bep_matches_single(world):
    from dpm_inputs import get_config
    from oracle import dpm
    ref = dpm.cfg1_outputs(get_config("cfg1"))["B"].T
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert np.array_equal(res[r], ref), r   # column sharding is exact (bit-identical columns)
