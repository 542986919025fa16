"""World-size-2/3 `gloo` runs of the theta-slab sharding on CPU, through the
library's C-ABI wherever it has no device work: the rank partition
(ea_theta_slab), the NCCL id handed from rank 0 to every rank
(ea_comm_unique_id -> ea_comm_init's input), the `better` merge
(ea_merge_topk).  Per rank, the C oracle stands in for the device search
over its slab; one all-gather; the merge == the single-process search_topk,
bit for bit, on every rank."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from paper_2112_05576_b200 import abi, api, parallel

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
        # the same exchange with the library's merge (ea_merge_topk, C-ABI)
        import torch
        rows = torch.from_numpy(parallel.pack(local, k))
        allrows = torch.empty((world * k, parallel.ROW), dtype=torch.float64)
        dist.all_gather_into_tensor(allrows, rows)
        merged_c = api.merge_topk(parallel.unpack(allrows.numpy()), k)
        # rank 0's NCCL id reaches every rank intact (the ea_comm_init input)
        cid = parallel.share_comm_id()
        ids = [None] * world
        dist.all_gather_object(ids, abi.comm_id_bytes(cid))
        q.put((rank, [(s.score, int(s.grid_index), s.pose.astuple()) for s in merged],
               [(s.score, int(s.grid_index), s.pose.astuple()) for s in merged_c],
               (it0, it1), len(set(ids)) == 1 and len(ids[0]) == abi.EA_COMM_ID_BYTES))
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
    got = [q.get(timeout=240) for _ in procs]
    res = {g[0]: g[1] for g in got}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc, m, f, grid = case(seed)
    full = orc.search_topk(m.points, f, grid, abi.ScoreParams(3), k)
    want = [(s.score, int(s.grid_index), s.pose.astuple()) for s in full]
    for r in range(world):
        assert res[r] == want
    slabs = sorted(g[3] for g in got)
    assert slabs[0][0] == 0 and slabs[-1][1] == orc.grid_counts(grid)[2]
    assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))
    for g in got:
        assert g[2] == want  # library merge
        assert g[4]          # one id on every rank


def test_slab_partition_covers_grid():
    """ea_theta_slab == the reference's block partition (search.cpp:116-120)."""
    for nt in (1, 5, 7, 720, 1440, 2 ** 40 + 3):
        for world in (1, 2, 3, 8, 16):
            slabs = [parallel.theta_slab(nt, r, world) for r in range(world)]
            assert slabs == [(nt * r // world, nt * (r + 1) // world) for r in range(world)]
            assert slabs[0][0] == 0 and slabs[-1][1] == nt
            assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))
    assert api.theta_slab(10, 3, 2) == (0, 0)  # rank out of range: empty


def test_comm_id_roundtrip():
    cid = api.comm_unique_id()
    raw = abi.comm_id_bytes(cid)
    assert len(raw) == abi.EA_COMM_ID_BYTES
    assert abi.comm_id_bytes(abi.comm_id_from_bytes(raw)) == raw


def test_pack_unpack_roundtrip():
    s = [abi.ScoredPose(0.5, 2 ** 40 + 3, abi.Pose(1.5, -2.25, 0.125))]
    back = parallel.unpack(parallel.pack(s, 3))
    assert len(back) == 1 and back[0].grid_index == 2 ** 40 + 3
    assert back[0].score == 0.5 and back[0].pose.astuple() == (1.5, -2.25, 0.125)


# ---- multi-model sharding: ea_plan_multi ---------------------------
def check_plan(items, thetas, world):
    """Every model's theta range is covered exactly once by contiguous slabs,
    one slab per (rank, model), ranks in range."""
    by_model = {}
    seen = set()
    for r, m, b, e, c in items:
        assert 0 <= r < world and b < e and c > 0
        assert (r, m) not in seen
        seen.add((r, m))
        by_model.setdefault(m, []).append((b, e))
    for m, nt in enumerate(thetas):
        sl = sorted(by_model.get(m, []))
        if nt == 0:
            assert not sl
            continue
        assert sl[0][0] == 0 and sl[-1][1] == nt
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8, 16])
def test_plan_multi_covers_and_balances(world):
    ntop = [11, 20, 35, 57, 75, 144, 210, 292]  # cfg5's top-level model sizes
    planes, thetas = [324 * 243] * 8, [720] * 8
    items = api.plan_multi(planes, thetas, ntop, world)
    check_plan(items, thetas, world)
    assert items == api.plan_multi(planes, thetas, ntop, world)  # deterministic
    load = [0.0] * world
    for r, m, b, e, c in items:
        load[r] += c
    ideal = sum(p * t * n for p, t, n in zip(planes, thetas, ntop)) / world
    # within the fixed per-search cost of one slab per model of the ideal
    assert max(load) <= ideal * 1.15 + 8 * 6.6e7
    # never worse than cutting every model into `world` slabs
    uniform = ideal + 8 * 6.6e7
    assert max(load) <= uniform * 1.0001


def test_plan_multi_edge_cases():
    assert api.plan_multi([], [], [], 4) == []
    items = api.plan_multi([100, 100], [3, 0], [5, 7], 8)  # fewer thetas than ranks; empty model
    check_plan(items, [3, 0], 8)
    assert all(m == 0 for _, m, _, _, _ in items) and len(items) <= 3
    from paper_2112_05576_b200.errors import InvalidArgument
    with pytest.raises(InvalidArgument):
        api.plan_multi([1], [1], [1], 0)


def multi_case(seed):
    from oracle.pyoracle import OracleC
    orc = OracleC()
    img, _, _, _ = orc.compose_scene(abi.SceneSpec(96, 80, "cross", 30, (40, 36, D(20)), 14,
                                                   seed))
    models = []
    for shape, size in (("l_bracket", 32), ("cross", 30), ("ring", 24)):
        models.append(orc.prepare_model(orc.render_template(shape, size)))
    f = orc.compute_gradients(img)
    grid = abi.PoseGrid(0, 95, 1, 0, 79, 1, 0.0, D(350), D(10))
    return orc, models, f, grid


def multi_worker(rank, world, port, seed, k, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc, models, f, grid = multi_case(seed)
        nx, ny, nt = orc.grid_counts(grid)
        n = len(models)
        items = api.plan_multi([nx * ny] * n, [nt] * n, [len(m.points) for m in models], world)
        rows = np.full((n * k, parallel.ROW), np.nan)
        for r, m, b, e, _ in items:  # this rank's (model, slab) items; oracle stands in
            if r == rank:
                part = orc.search_topk(models[m].points, f, grid, abi.ScoreParams(3), k,
                                       it_range=(b, e), threads=2)
                rows[m * k:(m + 1) * k] = parallel.pack(part, k)
        allrows = torch.empty((world * n * k, parallel.ROW), dtype=torch.float64)
        dist.all_gather_into_tensor(allrows, torch.from_numpy(rows))
        got = allrows.numpy().reshape(world, n, k, parallel.ROW)
        out = []
        for m in range(n):
            merged = api.merge_topk(parallel.unpack(got[:, m]), k)
            out.append([(s.score, int(s.grid_index)) for s in merged])
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,seed", [(2, 5, 1), (3, 4, 2)])
def test_multi_model_plan_gather_merge_equals_full(world, k, seed):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=multi_worker, args=(r, world, port, seed, k, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc, models, f, grid = multi_case(seed)
    want = [[(s.score, int(s.grid_index)) for s in
             orc.search_topk(m.points, f, grid, abi.ScoreParams(3), k)] for m in models]
    for r in range(world):
        assert res[r] == want
