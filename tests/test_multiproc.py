"""World-size-2 `gloo` runs of the theta-slab sharding (paper_2112_05576_b200
.parallel) on CPU: per-rank top-k over its slab (the C oracle stands in for
the device search here), one all-gather, `better` merge == the single-process
search_topk, bit for bit, on every rank."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from paper_2112_05576_b200 import abi, parallel

D = abi.deg_to_rad


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def case(seed):
    from oracle.pyoracle import OracleC
    orc = OracleC()
    img, tmpl, _, _ = orc.compose_scene(abi.SceneSpec(96, 80, "l_bracket", 40, (48, 40, D(33)),
                                                      12, seed))
    m = orc.prepare_model(tmpl)
    f = orc.compute_gradients(img)
    grid = abi.PoseGrid(0, 95, 1, 0, 79, 1, 0.0, D(355), D(5))
    return orc, m, f, grid


def worker(rank, world, port, seed, k, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc, m, f, grid = case(seed)
        nt = orc.grid_counts(grid)[2]
        it0, it1 = parallel.theta_slab(nt, rank, world)
        local = orc.search_topk(m.points, f, grid, abi.ScoreParams(3), k, it_range=(it0, it1),
                                threads=2)
        merged = parallel.gather_topk(local, k)
        q.put((rank, [(s.score, int(s.grid_index), s.pose.astuple()) for s in merged]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,seed", [(2, 5, 1), (2, 9, 2), (3, 4, 3)])
def test_theta_slabs_gather_merge_equals_full(world, k, seed):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, seed, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc, m, f, grid = case(seed)
    full = orc.search_topk(m.points, f, grid, abi.ScoreParams(3), k)
    want = [(s.score, int(s.grid_index), s.pose.astuple()) for s in full]
    for r in range(world):
        assert res[r] == want


def test_slab_partition_covers_grid():
    for nt in (1, 7, 720, 1440):
        for world in (1, 2, 3, 8):
            slabs = [parallel.theta_slab(nt, r, world) for r in range(world)]
            assert slabs[0][0] == 0 and slabs[-1][1] == nt
            assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))


def test_pack_unpack_roundtrip():
    s = [abi.ScoredPose(0.5, 2 ** 40 + 3, abi.Pose(1.5, -2.25, 0.125))]
    back = parallel.unpack(parallel.pack(s, 3))
    assert len(back) == 1 and back[0].grid_index == 2 ** 40 + 3
    assert back[0].score == 0.5 and back[0].pose.astuple() == (1.5, -2.25, 0.125)
