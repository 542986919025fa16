"""The multi-GPU data path of the C++ library (include/edgealign_b200.h,
"multi-GPU") on one B200: an NCCL communicator of world size 1 joined with
ea_comm_init, the device all-gather + `better` merge (ea_gather_rows_async),
the sharded detect (ea_detect_sharded: input broadcast, slab search,
all-gather, merge, root refinement, outcome broadcast) and its host-only
partition (ea_theta_slab).  Results must equal the single-GPU detect and the
CPU oracle bit for bit (reference run_search partition + merge,
search.cpp:116-139).  Several ranks on one GPU are not run (their kernels
would wait on one another); the rank logic at world 2/3 is covered on CPU by
tests/test_multiproc.py."""
import numpy as np
import pytest

from paper_2112_05576_b200 import abi, parallel

pytestmark = pytest.mark.gpu

D = abi.deg_to_rad


def keys(lst):
    return [(s.score, int(s.grid_index), s.pose.astuple()) for s in lst]


def scene(ea, **kw):
    img, tmpl, _, _ = ea.compose_scene(ea.SceneSpec(**kw))
    return img, tmpl


@pytest.fixture()
def comm_ctx(ea):
    """A fresh context joined to a world-1 NCCL communicator."""
    ctx = ea.Context(0)
    ctx.comm_init(0, 1, ea.comm_unique_id())
    assert ctx.comm_info() == (0, 1)
    yield ctx
    ctx.comm_destroy()
    assert not ctx.has_comm()
    ctx.close()


CASES = [
    dict(scene=dict(canvas_width=200, canvas_height=160, template_id="l_bracket",
                    template_size=56, true_pose=(96, 84, D(63)), clutter_segments=25,
                    clutter_seed=4, noise_sigma=1.0, noise_seed=2),
         grid=(0, 199, 4, 0, 159, 4, 0.0, D(357), D(3)), L=3, k=4),
    dict(scene=dict(canvas_width=320, canvas_height=240, template_id="l_bracket",
                    template_size=64, true_pose=(150, 110, D(200)), clutter_segments=30,
                    clutter_seed=5, noise_sigma=2.0, noise_seed=3,
                    illumination=(1.3, -10.0, 1.1)),
         grid=(0, 319, 4, 0, 239, 4, 0.0, D(358), D(2)), L=3, k=5),
    dict(scene=dict(canvas_width=256, canvas_height=256, template_id="rectangle",
                    template_size=64, true_pose=(100, 60, D(30))),
         grid=(40, 216, 8, 40, 216, 8, 0.0, D(88), D(4)), L=2, k=5),
    # no refinement level: the merged seed is the answer
    dict(scene=dict(canvas_width=96, canvas_height=96, template_id="cross", template_size=32,
                    true_pose=(48, 48, 0.0)),
         grid=(24, 72, 2, 24, 72, 2, 0.0, 0.0, 1.0), L=1, k=5),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_detect_sharded_world1_equals_detect_and_oracle(ea, oracle, comm_ctx, case):
    c = CASES[case]
    img, tmpl = scene(ea, **c["scene"])
    cfg = ea.SearchConfig(grid=ea.PoseGrid(*c["grid"]), num_levels=c["L"],
                          score_params=ea.ScoreParams(3), topk=c["k"])
    det = ea.Detector(tmpl, cfg, comm_ctx)
    got = det.detect_sharded(img)
    again = det.detect_sharded(img)  # cached plane / tables path
    single = det.detect(img)
    assert got.key() == single.key() == again.key()
    want = oracle.coarse_to_fine(oracle.build_pyramid(tmpl, c["L"]),
                                 oracle.build_pyramid(img, c["L"]), cfg)
    assert got.key() == want.key()
    # search_levels_sharded on the working image already set
    assert ea.search_levels_sharded(det.levels, cfg).key() == want.key()


def test_gather_rows_library_nccl_world1(ea, comm_ctx):
    """ea_gather_rows_async (NCCL all-gather + device merge, inside the
    library) on one rank == the rank's own rows == ea_search_top_slab."""
    import torch
    img, tmpl = scene(ea, canvas_width=160, canvas_height=128, template_id="l_bracket",
                      template_size=48, true_pose=(80, 64, D(20)), clutter_segments=10,
                      clutter_seed=3)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 159, 2, 0, 127, 2, 0.0, D(355), D(5)),
                          num_levels=2, score_params=ea.ScoreParams(3), topk=5)
    det = ea.Detector(tmpl, cfg, comm_ctx)
    det.levels.set_image(img)
    stream = torch.cuda.Stream()
    comm_ctx.set_stream(stream.cuda_stream)
    try:
        rows = torch.empty((5, 5), dtype=torch.float64, device="cuda")
        ea.search_top_slab_async(det.levels, cfg, 0, 72, rows.data_ptr())
        merged = parallel.gather_rows_device(rows, 5, comm_ctx)
        stream.synchronize()
        overflowed, _ = ea.async_status(comm_ctx)
        assert not overflowed
    finally:
        comm_ctx.set_stream(None)
    want = ea.search_top_slab(det.levels, cfg, 0, 72)
    assert keys(parallel.unpack(merged.cpu().numpy())) == keys(want)
    assert keys(parallel.unpack(rows.cpu().numpy())) == keys(want)


def test_gather_rows_needs_comm(ea):
    import torch
    ctx = ea.Context(0)
    try:
        rows = torch.zeros((5, 5), dtype=torch.float64, device="cuda")
        with pytest.raises(ea.InvalidArgument, match="no communicator"):
            ea.gather_rows_async(ctx, rows.data_ptr(), 5, rows.data_ptr())
    finally:
        ctx.close()


def test_empty_slab_rows_are_empty_after_a_search(ea):
    """An empty theta slab (more ranks than thetas) writes k NaN rows, never
    the previous search's top k (stale n_out)."""
    import torch
    img, tmpl = scene(ea, canvas_width=160, canvas_height=128, template_id="l_bracket",
                      template_size=48, true_pose=(80, 64, D(20)), clutter_segments=10,
                      clutter_seed=3)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 159, 2, 0, 127, 2, 0.0, D(355), D(5)),
                          num_levels=2, score_params=ea.ScoreParams(3), topk=5)
    det = ea.Detector(tmpl, cfg)
    det.levels.set_image(img)
    rows = torch.empty((5, 5), dtype=torch.float64, device="cuda")
    ea.search_top_slab_async(det.levels, cfg, 0, 72, rows.data_ptr())
    ea.async_status(det.ctx)
    assert not np.isnan(rows.cpu().numpy()[:, 0]).any()
    for a, b in ((10, 10), (72, 72), (80, 90), (9, 3)):
        ea.search_top_slab_async(det.levels, cfg, a, b, rows.data_ptr())
        ea.async_status(det.ctx)
        assert np.isnan(rows.cpu().numpy()[:, 0]).all(), (a, b)
        assert ea.search_top_slab(det.levels, cfg, a, b) == []
    # and the next real search is unaffected
    ea.search_top_slab_async(det.levels, cfg, 0, 72, rows.data_ptr())
    ea.async_status(det.ctx)
    assert keys(parallel.unpack(rows.cpu().numpy())) == keys(ea.search_top_slab(det.levels, cfg, 0, 72))


@pytest.mark.parametrize("n", [3072, 3200, 8192])
def test_merge_rows_many(ea, n):
    """More rows than the 48 KB default dynamic shared memory holds (ADVICE
    r01: merge_rows_kernel did not opt in): the merge == a host sort by
    `better`, including tied scores broken by index and NaN (empty) rows."""
    import torch
    rng = np.random.default_rng(n)
    k = 7
    rows = np.zeros((n, 5))
    rows[:, 0] = rng.integers(0, 50, size=n) / 64.0
    rows[:, 1] = rng.permutation(10 * n)[:n]
    rows[:, 2:] = rng.normal(size=(n, 3))
    rows[rng.random(n) < 0.2, 0] = np.nan
    d_in = torch.from_numpy(rows).cuda()
    d_out = torch.empty((k, 5), dtype=torch.float64, device="cuda")
    ctx = ea.default_context()
    ea.merge_rows_async(ctx, d_in.data_ptr(), n, k, d_out.data_ptr())
    ctx.synchronize()
    want = parallel.merge(parallel.unpack(rows), k)
    assert keys(parallel.unpack(d_out.cpu().numpy())) == keys(want)


def test_detect_multi_sharded_world1(ea, oracle, comm_ctx):
    """ea_detect_multi_sharded (plan, input broadcast, per-item slab searches,
    one all-gather of every model's rows, per-model merge, root refinement,
    outcome broadcast) on a world-1 communicator == detect_multi == oracle,
    twice (cached plane and tables), on a region-tiled top level."""
    stamps = [("l_bracket", 64, (150.0, 130.0, D(40))), ("cross", 96, (460.0, 140.0, D(15))),
              ("ring", 80, (170.0, 350.0, 0.0)), ("rectangle", 72, (470.0, 340.0, D(200)))]
    spec = ea.SceneSpec(640, 480, "rectangle", 0, (0, 0, 0), 60, 5, None, (1.1, 4.0, 1.0), 1.5, 9)
    img = ea.compose_multi(spec, stamps)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 639, 2, 0, 479, 2, 0.0, D(350), D(10)),
                          num_levels=2, score_params=ea.ScoreParams(3), topk=3)
    tmpls = [ea.render_template(t, s) for t, s, _ in stamps]
    dets = [ea.Detector(t, cfg, comm_ctx) for t in tmpls]
    got = ea.detect_multi_sharded(dets, img)
    again = ea.detect_multi_sharded(dets, img)
    single = ea.detect_multi(dets, img)
    wp = oracle.build_pyramid(img, 2)
    for t, a, b, c in zip(tmpls, got, again, single):
        want = oracle.coarse_to_fine(oracle.build_pyramid(t, 2), wp, cfg)
        assert a.key() == b.key() == c.key() == want.key()


def test_detect_multi_sharded_lattice_world1(ea, oracle, comm_ctx):
    """Same on a small (shared-memory) top level with three refinement levels."""
    stamps = [("l_bracket", 48, (70.0, 60.0, D(33))), ("cross", 40, (150.0, 100.0, D(80)))]
    spec = ea.SceneSpec(224, 160, "rectangle", 0, (0, 0, 0), 20, 3, None, (1.0, 0.0, 1.0), 0.0, 0)
    img = ea.compose_multi(spec, stamps)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 223, 4, 0, 159, 4, 0.0, D(357), D(3)),
                          num_levels=3, score_params=ea.ScoreParams(3), topk=4)
    tmpls = [ea.render_template(t, s) for t, s, _ in stamps]
    dets = [ea.Detector(t, cfg, comm_ctx) for t in tmpls]
    got = ea.detect_multi_sharded(dets, img)
    wp = oracle.build_pyramid(img, 3)
    for t, a in zip(tmpls, got):
        assert a.key() == oracle.coarse_to_fine(oracle.build_pyramid(t, 3), wp, cfg).key()


@pytest.mark.parametrize("k", [1, 5, 8])
def test_blank_frame_async_and_sync(ea, k):
    """A featureless 1280x1024 frame (every pose scores exactly 0):
    the device-resident slab search no longer floods the band -- exact-zero
    tiles contribute only their first k poses -- and returns the reference's
    answer: the k smallest grid indices, score 0 (better: ties by index)."""
    import torch
    blank = np.full((1024, 1280), 117.0)
    tmpl = ea.render_template("l_bracket", 200)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 1279, 8, 0, 1023, 8, 0.0, D(359.5), D(0.5)),
                          num_levels=4, score_params=ea.ScoreParams(3), topk=k)
    det = ea.Detector(tmpl, cfg)
    det.levels.set_image(blank)
    rows = torch.empty((k, 5), dtype=torch.float64, device="cuda")
    ea.search_top_slab_async(det.levels, cfg, 0, 720, rows.data_ptr())
    overflowed, _ = ea.async_status(det.ctx)
    assert not overflowed
    got = parallel.unpack(rows.cpu().numpy())
    tg = ea.PoseGrid(0, 1279 / 8, 1, 0, 1023 / 8, 1, 0.0, D(359.5), D(0.5))
    want = [(0.0, i, ea.pose_at(tg, i).astuple()) for i in range(k)]
    assert [(s.score, int(s.grid_index), s.pose.astuple()) for s in got] == want
    sync = ea.search_top_slab(det.levels, cfg, 0, 720)
    assert keys(sync) == keys(got)
    # k per zero tile (at most 10 x 4 lattice tiles of 16 x 64 poses per
    # theta here), not every one of the 1.47e7 poses
    assert det.ctx.stats()["candidates"] <= 720 * 40 * k
    out = det.detect(blank)
    assert not out.found and out.score == 0.0


@pytest.mark.slow
def test_grid_over_2_32_poses_chunked(ea, oracle):
    """A pose grid of more than 2^32 poses (the reference indexes poses with
    size_t, search.cpp:105-106): searched in theta chunks whose top-k lists
    are `better`-merged.  The sync search, the device-resident slab rows and
    the detect path agree with each other and with the merge of explicit
    sub-slab searches; the returned scores are the oracle's pose scores."""
    import torch
    rng = np.random.default_rng(42)
    img = rng.integers(0, 256, size=(72, 72)).astype(np.float64)
    f = oracle.compute_gradients(img)
    m = oracle.extract_edge_model(oracle.compute_gradients(
        rng.integers(0, 256, size=(6, 6)).astype(np.float64)), (0.0, 0.0), 0)
    nt = (2 ** 32) // (64 * 64) + 50_000  # > 2^32 poses
    dt = 2e-6
    grid = ea.PoseGrid(4, 67, 1, 4, 67, 1, 0.0, (nt - 1) * dt, dt)
    nx, ny, ntt = ea.grid_counts(grid)
    assert nx * ny * ntt > 2 ** 32
    params = ea.ScoreParams(3)
    k = 5
    full = ea.search_topk(m, f, grid, params, k=k)
    cuts = [0, 300_001, 700_000, ntt // 2 + 17, ntt]
    parts = []
    for a, b in zip(cuts, cuts[1:]):
        parts += ea.search_topk_slab(m, f, grid, params, k, a, b)
    assert keys(full) == keys(ea.merge_topk(parts, k))
    for s in full:
        want, _ = oracle.pose_score(m.points, s.pose.astuple(), f, params)
        assert s.score == want


def test_bench_rows_suite(ea):
    """cmd_bench's rows on the device: samples x backends x reps rows, all
    backends (every kind runs on the device) agreeing on the pose."""
    samples = []
    for i in range(2):
        img, tmpl = scene(ea, canvas_width=160, canvas_height=128, template_id="cross",
                          template_size=40, true_pose=(70 + 10 * i, 60, D(15 * i)),
                          clutter_segments=6, clutter_seed=i)
        samples.append((f"s{i}", tmpl, img))
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 159, 2, 0, 127, 2, 0.0, D(355), D(5)),
                          num_levels=2, score_params=ea.ScoreParams(3))
    rows = ea.bench_rows(samples, reps=2, warmup=1, backends=("serial", "parallel", "cuda"),
                         config=cfg)
    assert len(rows) == 2 * 3 * 2
    assert all(r["elapsed_ms"] > 0 for r in rows)
    text = ea.bench_csv(rows)
    assert text.splitlines()[0] == "sample,backend,workers,run,elapsed_ms"
