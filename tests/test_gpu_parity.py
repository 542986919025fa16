"""CUDA path vs the CPU oracle (oracle/edgealign_oracle.c, pinned to the
reference in tests/test_oracle_ref.py): bit-exact poses, indices and scores.

Cases follow the reference's own tests (proj/tests/test_search.cpp,
test_similarity.cpp, test_edge_model.cpp, test_image.cpp) plus the lattice /
general screening paths, theta slabs and the BASELINE configs' geometry.
"""
import math

import numpy as np
import pytest

from paper_2112_05576_b200 import abi

pytestmark = pytest.mark.gpu

D = abi.deg_to_rad


def rand_image(rng, w, h, real=False):
    if real:
        return rng.uniform(-40.0, 300.0, size=(h, w))
    return rng.integers(0, 256, size=(h, w)).astype(np.float64)


def rand_model(oracle, rng, size):
    f = oracle.compute_gradients(rand_image(rng, size, size))
    return oracle.extract_edge_model(f, (0.0, 0.0), 0)


def keys(lst):
    return [(s.score, int(s.grid_index), s.pose.astuple()) for s in lst]


# ---- field side ----------------------------------------------------------------------
@pytest.mark.parametrize("w,h", [(3, 3), (4, 5), (17, 9), (64, 48), (161, 123), (640, 480)])
def test_gradients_bit_exact(ea, oracle, w, h):
    rng = np.random.default_rng(w * 1000 + h)
    for real in (False, True):
        img = rand_image(rng, w, h, real)
        got = ea.compute_gradients(img)
        want = oracle.compute_gradients(img)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)


def test_gradient_kats(ea):
    # test_edge_model.cpp:50-92: constant -> 0; vertical step -> gx = 32
    f = ea.compute_gradients(np.full((7, 9), 123.25))
    assert not f.gx.any() and not f.gy.any() and not f.mag.any()
    img = np.zeros((7, 9))
    img[:, 4:] = 8.0
    f = ea.compute_gradients(img)
    assert (f.gx[1:6, 3] == 32).all() and (f.gx[1:6, 4] == 32).all()
    assert (f.gy[1:6, 3] == 0).all() and (f.mag[1:6, 3] == 32).all()
    with pytest.raises(ea.SizeError):
        ea.compute_gradients(np.zeros((8, 2)))


@pytest.mark.parametrize("w,h,levels", [(2, 2, 1), (5, 5, 1), (812, 617, 3), (1280, 1024, 4),
                                        (2592, 1944, 5), (33, 17, 2)])
def test_pyramid_bit_exact(ea, oracle, w, h, levels):
    rng = np.random.default_rng(7)
    img = rand_image(rng, w, h, real=True)
    if levels <= oracle.max_pyramid_levels(w, h):
        got = ea.build_pyramid(img, levels)
        want = oracle.build_pyramid(img, levels)
        assert [g.shape for g in got] == [x.shape for x in want]
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
    assert np.array_equal(ea.downsample(img), oracle.downsample(img))


def test_pyramid_errors(ea):
    with pytest.raises(ea.SizeError, match="maximum feasible level count is 2"):
        ea.build_pyramid(np.zeros((16, 16)), 4)
    with pytest.raises(ea.SizeError):
        ea.downsample(np.zeros((5, 1)))
    assert ea.max_pyramid_levels(16, 16) == 2


# ---- similarity ---------------------------------------------------------------------
def test_point_vote_kats(ea):
    # test_similarity.cpp:45-81
    def field(w, h, sets):
        gx, gy = np.zeros((h, w)), np.zeros((h, w))
        for (x, y, a, b) in sets:
            gx[y, x], gy[y, x] = a, b
        return (gx, gy, np.sqrt(gx * gx + gy * gy))

    P = ea.ScoreParams
    assert ea.point_vote(1, 0, field(7, 7, [(3, 3, 5, 0)]), 3, 3, P(3)) == pytest.approx(1.0, abs=1e-12)
    assert ea.point_vote(1, 0, field(7, 7, []), 3, 3, P(3)) == 0.0
    f = field(7, 7, [(3, 3, -5, 0), (4, 3, 1e-4, 0)])
    assert ea.point_vote(1, 0, f, 3, 3, P(3)) == pytest.approx(1.0, abs=1e-12)
    assert ea.point_vote(1, 0, f, 3, 3, P(1)) == pytest.approx(-1.0, abs=1e-12)
    z = field(5, 5, [])
    assert ea.point_vote(0, 1, z, 40, 40, P(3)) == 0.0
    assert ea.point_vote(0, 1, z, -9, 2, P(3)) == 0.0
    assert ea.point_vote(1, 0, field(5, 5, [(2, 2, -7, 0)]), 2, 2,
                         P(1, abi.POLARITY_IGNORE)) == pytest.approx(1.0)
    with pytest.raises(ea.InvalidArgument, match="neighborhood must be odd"):
        ea.point_vote(1, 0, z, 2, 2, P(2))
    with pytest.raises(ea.InvalidArgument, match="eps_mag must be positive"):
        ea.point_vote(1, 0, z, 2, 2, P(3, 0, 0.0))


def test_rotate_model_bit_exact(ea, oracle):
    rng = np.random.default_rng(5)
    m = rand_model(oracle, rng, 14)
    for theta in [0.0, 0.3, -2.0, D(30), D(359.75), 7.1]:
        got = ea.rotate_model(m, theta)
        want = oracle.rotate_model(m.points, theta)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)


def test_pose_score_bit_exact(ea, oracle):
    rng = np.random.default_rng(37)
    m = oracle.prepare_model(oracle.render_template("cross", 32))
    f = oracle.compute_gradients(rand_image(rng, 48, 48))
    for trial in range(60):
        pose = (rng.uniform(-10, 58), rng.uniform(-10, 58), rng.uniform(-3.2, 3.2))
        for params in (ea.ScoreParams(1), ea.ScoreParams(3), ea.ScoreParams(5),
                       ea.ScoreParams(3, abi.POLARITY_IGNORE)):
            assert ea.pose_score(m, pose, f, params) == oracle.pose_score(m.points, pose, f, params)
    v, n = ea.pose_score(m, (500, 500, 0.3), f, ea.ScoreParams(3))
    assert v == 0.0 and n == 0


# ---- top-level search ------------------------------------------------------------------
SEARCH_CASES = [
    # (model size, field w, h, grid, nb, polarity)  -- test_search.cpp:55-98 shapes
    (8, 32, 32, (4, 27, 1, 4, 27, 1, 0.0, D(30), D(15)), 3, 0),
    (10, 32, 32, (4, 27, 1, 4, 27, 1, 0.0, D(30), D(15)), 1, 0),
    (12, 40, 40, (0, 39, 1, 0, 39, 1, 0.0, D(20), D(10)), 3, 0),
    (14, 32, 32, (4, 27, 1, 4, 27, 1, 0.0, D(30), D(15)), 5, 0),
    (12, 40, 40, (0, 39, 1, 0, 39, 1, 0.0, D(20), D(10)), 3, 1),
    (12, 40, 40, (-6, 45, 1, -7, 44, 1, 0.0, D(359), D(1)), 3, 0),   # off-image overhang
    (10, 30, 30, (5, 24, 2, 5, 24, 3, 0.0, D(10), D(5)), 3, 0),      # integer, non-unit step
    (10, 30, 30, (0.5, 24.5, 1, 2.25, 20, 0.75, 0.1, 0.9, 0.2), 3, 0),  # general grid
    (20, 64, 48, (0, 63, 1, 0, 47, 1, 0.0, D(355), D(5)), 3, 0),
]


@pytest.mark.parametrize("case", range(len(SEARCH_CASES)))
def test_search_topk_bit_exact(ea, oracle, case):
    size, w, h, g, nb, pol = SEARCH_CASES[case]
    rng = np.random.default_rng(100 + case)
    m = rand_model(oracle, rng, size)
    f = oracle.compute_gradients(rand_image(rng, w, h))
    grid = ea.PoseGrid(*g)
    params = ea.ScoreParams(nb, pol)
    for k in (1, 5, 17):
        got = ea.search_topk(m, f, grid, params, k=k)
        want = oracle.search_topk(m.points, f, grid, params, k)
        assert keys(got) == keys(want)
    det = ea.exhaustive_search(m, f, grid, params)
    ref = oracle.exhaustive_search(m.points, f, grid, params)
    assert (det.score, det.grid_index) == (ref.score, ref.grid_index)


def test_search_uploaded_field_with_border(ea, oracle):
    """A field whose outer ring votes (not from compute_gradients) must take
    the exactly-clipped general path."""
    rng = np.random.default_rng(3)
    m = rand_model(oracle, rng, 10)
    gx = rng.normal(size=(30, 34))
    gy = rng.normal(size=(30, 34))
    f = (gx, gy, np.sqrt(gx * gx + gy * gy))
    grid = ea.PoseGrid(0, 33, 1, 0, 29, 1, 0.0, D(40), D(10))
    got = ea.search_topk(m, f, grid, ea.ScoreParams(3), k=5)
    assert keys(got) == keys(oracle.search_topk(m.points, f, grid, ea.ScoreParams(3), 5))
    assert ea.default_context().stats()["screen_path"] == 2


def test_search_flat_field_ties(ea, oracle):
    """All scores 0: the top k are the k smallest indices (search.cpp:36-41)."""
    m = oracle.prepare_model(oracle.render_template("rectangle", 32))
    z = np.zeros((40, 40))
    f = (z, z, z)
    grid = ea.PoseGrid(0, 39, 1, 0, 39, 1, 0.0, D(20), D(10))
    got = ea.search_topk(m, f, grid, ea.ScoreParams(3), k=7)
    assert keys(got) == keys(oracle.search_topk(m.points, f, grid, ea.ScoreParams(3), 7))
    assert [int(s.grid_index) for s in got] == list(range(7))


def test_search_k_exceeds_grid(ea, oracle):
    rng = np.random.default_rng(11)
    m = rand_model(oracle, rng, 10)
    f = oracle.compute_gradients(rand_image(rng, 20, 20))
    grid = ea.PoseGrid(3, 5, 1, 4, 4, 1, 0.0, 0.2, 0.1)
    got = ea.search_topk(m, f, grid, ea.ScoreParams(3), k=50)
    want = oracle.search_topk(m.points, f, grid, ea.ScoreParams(3), 50)
    assert len(got) == 9 and keys(got) == keys(want)


def test_search_errors(ea, oracle):
    rng = np.random.default_rng(12)
    m = rand_model(oracle, rng, 10)
    f = oracle.compute_gradients(rand_image(rng, 20, 20))
    grid = ea.PoseGrid(0, 19, 1, 0, 19, 1, 0.0, 0.0, 1.0)
    with pytest.raises(ea.InvalidArgument, match="topk must be >= 1"):
        ea.search_topk(m, f, grid, ea.ScoreParams(3), k=0)
    empty = ea.EdgeModel(np.zeros((0, 5)))
    with pytest.raises(ea.InvalidArgument, match="search needs a nonempty model"):
        ea.search_topk(empty, f, grid, ea.ScoreParams(3), k=1)
    with pytest.raises(ea.InvalidArgument, match="steps must be positive"):
        ea.search_topk(m, f, ea.PoseGrid(0, 1, 0.0, 0, 1, 1, 0, 1, 1), ea.ScoreParams(3), k=1)
    with pytest.raises(ea.BudgetError, match="900"):
        ea.score_map(m, f, ea.PoseGrid(0, 29, 1, 0, 29, 1, 0, 0, 1), ea.ScoreParams(1), 100)


def test_score_map_bit_exact(ea, oracle):
    rng = np.random.default_rng(67)
    m = rand_model(oracle, rng, 10)
    f = oracle.compute_gradients(rand_image(rng, 30, 30))
    for g in [(5, 24, 1, 5, 24, 1, 0.0, D(10), D(5)), (7, 7, 1, 7, 7, 1, 0.1, 0.1, 1.0),
              (0.25, 20, 1.5, 1, 22, 2.5, -0.5, 0.5, 0.25)]:
        grid = ea.PoseGrid(*g)
        got = ea.score_map(m, f, grid, ea.ScoreParams(3), 1 << 20)
        want = oracle.score_map(m.points, f, grid, ea.ScoreParams(3), 1 << 20)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("nb,pol,general", [(3, 0, False), (1, 0, False), (5, 0, False),
                                            (3, 1, False), (3, 0, True), (7, 1, True)])
def test_screen_bound(ea, oracle, nb, pol, general):
    """|S_f - S| <= delta for every pose (the premise of exactness)."""
    rng = np.random.default_rng(nb * 10 + pol)
    tm = oracle.prepare_model(oracle.render_template("l_bracket", 48))
    f = oracle.compute_gradients(rand_image(rng, 40, 36, real=True))
    if general:
        grid = ea.PoseGrid(-3.5, 40, 1, -2.5, 38, 1, 0.0, D(350), D(10))
    else:
        grid = ea.PoseGrid(-4, 43, 1, -3, 38, 1, 0.0, D(350), D(10))
    params = ea.ScoreParams(nb, pol)
    sf, delta = ea.screen_map(tm, f, grid, params)
    s = oracle.score_map(tm.points, f, grid, params, 1 << 30)
    err = np.abs(sf.astype(np.float64) - s).max()
    assert err <= delta, (err, delta)
    assert delta < 2e-6


REGION_CASES = [
    # (model, size, field w, h, grid, nb, polarity): top planes larger than
    # shared memory -> region-tiled lattice kernel (screen_path 3)
    ("l_bracket", 40, 400, 330, (0, 399, 1, 0, 329, 1, 0.0, D(330), D(30)), 3, 0),
    ("rectangle", 64, 420, 300, (-12, 431, 1, -9, 310, 1, 0.1, D(200), D(20)), 3, 0),
    ("ring", 24, 380, 380, (0, 379, 1, 0, 379, 1, 0.0, D(350), D(50)), 1, 0),
    ("cross", 48, 400, 320, (3, 396, 1, 2, 317, 1, 0.0, D(340), D(20)), 5, 0),
    ("l_bracket", 64, 360, 360, (0, 359, 1, 0, 359, 1, 0.0, D(300), D(60)), 3, 1),
    # plane fits shared memory only with shrunk zero columns -> clamping variant
    ("l_bracket", 72, 300, 85, (0, 299, 1, 0, 84, 1, 0.0, D(330), D(30)), 3, 0),
    # halo region of a 96 px model: general kernel, or region kernel when it fits
    ("l_bracket", 96, 360, 360, (0, 359, 1, 0, 359, 1, 0.0, D(300), D(60)), 3, 0),
]


@pytest.mark.parametrize("case", range(len(REGION_CASES)))
def test_region_search_bit_exact(ea, oracle, case):
    shape, size, w, h, g, nb, pol = REGION_CASES[case]
    rng = np.random.default_rng(300 + case)
    tm = oracle.prepare_model(oracle.render_template(shape, size))
    f = oracle.compute_gradients(rand_image(rng, w, h, real=case % 2 == 1))
    grid = ea.PoseGrid(*g)
    params = ea.ScoreParams(nb, pol)
    for k in (1, 9):
        got = ea.search_topk(tm, f, grid, params, k=k)
        path = ea.default_context().stats()["screen_path"]
        # a 96 px model's halo region fits shared memory only without the
        # histogram (top-list mode, k <= 8) and with 4-row strips (twins)
        assert path == (1 if h < 100 else 3) if size <= 90 else path in (2, 3)
        want = oracle.search_topk(tm.points, f, grid, params, k)
        assert keys(got) == keys(want)


GEOMETRY_SWEEP = [
    # (shape, size, w, h, grid): planes around the shared-memory limit for
    # 8- and 4-row strips, very wide and very thin fields and grids (one
    # translation row, one column), grids overhanging the field
    ("rectangle", 40, 280, 96, None),
    ("l_bracket", 56, 310, 90, None),
    ("rectangle", 40, 330, 80, None),
    ("l_bracket", 48, 512, 50, None),
    ("cross", 40, 900, 24, None),
    ("rectangle", 32, 1500, 12, None),
    ("l_bracket", 40, 1200, 40, (0, 1199, 1, 20, 20, 1, 0.0, D(270), D(90))),
    ("rectangle", 40, 64, 900, (30, 30, 1, 0, 899, 1, 0.0, D(270), D(90))),
    ("ring", 30, 200, 150, (-40, 239, 1, -30, 179, 1, 0.0, D(300), D(60))),
    # integer strides > 1 on a plane too large for shared memory (region
    # kernel, strided emit) and on a fitting one
    ("l_bracket", 48, 640, 480, (0, 639, 3, 0, 479, 3, 0.0, D(270), D(90))),
    ("rectangle", 40, 300, 200, (1, 298, 2, 2, 197, 4, 0.0, D(270), D(90))),
]


@pytest.mark.parametrize("case", range(len(GEOMETRY_SWEEP)))
def test_search_geometry_sweep(ea, oracle, case):
    """Field and grid shapes at the lattice kernels' limits (plane bytes vs
    the shared-memory budget, padding shrunk or not, region tiling, warp
    tiles much wider or taller than the grid) == the oracle."""
    shape, size, w, h, g = GEOMETRY_SWEEP[case]
    rng = np.random.default_rng(4000 + case)
    tm = oracle.prepare_model(oracle.render_template(shape, size))
    f = oracle.compute_gradients(rand_image(rng, w, h, real=case % 2 == 0))
    grid = ea.PoseGrid(*(g or (0, w - 1, 1, 0, h - 1, 1, 0.0, D(270), D(90))))
    params = ea.ScoreParams(3)
    for k in (1, 5, 9):
        got = ea.search_topk(tm, f, grid, params, k=k)
        want = oracle.search_topk(tm.points, f, grid, params, k)
        assert keys(got) == keys(want), (k, ea.default_context().stats()["screen_path"])


@pytest.mark.parametrize("nb,pol", [(3, 0), (5, 1), (1, 0)])
def test_region_screen_bound(ea, oracle, nb, pol):
    rng = np.random.default_rng(40 + nb)
    tm = oracle.prepare_model(oracle.render_template("l_bracket", 56))
    f = oracle.compute_gradients(rand_image(rng, 300, 420, real=True))
    grid = ea.PoseGrid(-20, 310, 1, -15, 430, 1, 0.2, D(300), D(60))
    params = ea.ScoreParams(nb, pol)
    sf, delta = ea.screen_map(tm, f, grid, params)
    assert ea.default_context().stats()["screen_path"] == 3
    s = oracle.score_map(tm.points, f, grid, params, 1 << 30)
    err = np.abs(sf.astype(np.float64) - s).max()
    assert err <= delta, (err, delta)


@pytest.mark.parametrize("shape,size,w,h", [("rectangle", 32, 60, 50), ("ring", 24, 48, 48),
                                             ("ring", 96, 400, 320)])
def test_flagged_thetas_exact(ea, oracle, shape, size, w, h):
    """Half-integer model coordinates at 90/180/270 deg give rounding-ambiguous
    lattice offsets (cos 90 deg != 0 in fp64): those thetas go through the
    general kernel, the rest through the lattice (or region) kernel, and
    the screening bound stays two-sided, so the band stays narrow."""
    rng = np.random.default_rng(size + w)
    pts = np.array(oracle.prepare_model(oracle.render_template(shape, size)).points)
    pts[:, :2] = np.floor(pts[:, :2]) + 0.5  # half-integer coordinates (as pyramid models get)
    tm = ea.EdgeModel(pts)
    f = oracle.compute_gradients(rand_image(rng, w, h, real=True))
    grid = ea.PoseGrid(0, w - 1, 1, 0, h - 1, 1, 0.0, D(355), D(5))
    params = ea.ScoreParams(3)
    got = ea.search_topk(tm, f, grid, params, k=5)
    st = ea.default_context().stats()
    assert st["flagged_points"] > 0 and st["screen_path"] in (1, 3)
    assert st["candidates"] < 2000
    assert keys(got) == keys(oracle.search_topk(tm.points, f, grid, params, 5))
    if w * h <= 3000:
        sf, delta = ea.screen_map(tm, f, grid, params)
        s = oracle.score_map(tm.points, f, grid, params, 1 << 30)
        assert np.abs(sf.astype(np.float64) - s).max() <= delta


def test_theta_slabs_merge_to_full(ea, oracle):
    """Theta-sharded search + `better` merge == the full search (the
    multi-GPU exchange, search.cpp:116-139)."""
    rng = np.random.default_rng(21)
    m = oracle.prepare_model(oracle.render_template("l_bracket", 40))
    f = oracle.compute_gradients(rand_image(rng, 48, 40))
    grid = ea.PoseGrid(0, 47, 1, 0, 39, 1, 0.0, D(357), D(3))
    params = ea.ScoreParams(3)
    full = ea.search_topk(m, f, grid, params, k=5)
    nt = ea.grid_counts(grid)[2]
    for G in (2, 3, 8):
        parts = []
        for g in range(G):
            parts += ea.search_topk_slab(m, f, grid, params, 5, nt * g // G, nt * (g + 1) // G)
        assert keys(ea.merge_topk(parts, 5)) == keys(full)


# ---- coarse to fine ------------------------------------------------------------------------
def scene(ea, **kw):
    spec = ea.SceneSpec(**kw)
    img, tmpl, pose, occ = ea.compose_scene(spec)
    return img, tmpl


C2F_CASES = [
    # test_search.cpp:162-262 geometries
    dict(scene=dict(canvas_width=96, canvas_height=96, template_id="cross", template_size=32,
                    true_pose=(48, 48, 0.0)),
         cfg=dict(grid=(24, 72, 2, 24, 72, 2, 0.0, 0.0, 1.0), num_levels=1)),
    dict(scene=dict(canvas_width=256, canvas_height=256, template_id="rectangle",
                    template_size=64, true_pose=(100, 60, D(30))),
         cfg=dict(grid=(40, 216, 8, 40, 216, 8, 0.0, D(88), D(4)), num_levels=2, min_score=0.4)),
    dict(scene=dict(canvas_width=160, canvas_height=160, template_id="l_bracket",
                    template_size=48, true_pose=(80, 76, D(22)), clutter_segments=14,
                    clutter_seed=99),
         cfg=dict(grid=(40, 120, 6, 40, 120, 6, 0.0, D(45), D(5)), num_levels=2, topk=6)),
    dict(scene=dict(canvas_width=320, canvas_height=240, template_id="l_bracket",
                    template_size=64, true_pose=(150, 110, D(200)), clutter_segments=30,
                    clutter_seed=5, noise_sigma=2.0, noise_seed=3,
                    illumination=(1.3, -10.0, 1.1)),
         cfg=dict(grid=(0, 319, 4, 0, 239, 4, 0.0, D(358), D(2)), num_levels=3)),
]


@pytest.mark.parametrize("case", range(len(C2F_CASES)))
def test_coarse_to_fine_bit_exact(ea, oracle, case):
    c = C2F_CASES[case]
    img, tmpl = scene(ea, **c["scene"])
    cfgd = dict(c["cfg"])
    L = cfgd["num_levels"]
    cfg = ea.SearchConfig(grid=ea.PoseGrid(*cfgd.pop("grid")), score_params=ea.ScoreParams(3),
                          **cfgd)
    tp, wp = oracle.build_pyramid(tmpl, L), oracle.build_pyramid(img, L)
    want = oracle.coarse_to_fine(tp, wp, cfg)
    got = ea.coarse_to_fine(tp, wp, cfg)
    assert got.key() == want.key()
    det = ea.Detector(tmpl, cfg).detect(img)
    assert det.key() == want.key()


C2F_SWEEP = [
    # (template, size, canvas, pose, L, grid step at level 0, dtheta, topk,
    #  refine_radius, nb, polarity)
    ("l_bracket", 48, (200, 160), (97, 81, 33), 3, 4, 3, 1, 1, 3, 0),
    ("cross", 40, (190, 150), (90, 70, 10), 2, 2, 5, 8, 2, 5, 0),
    ("rectangle", 56, (230, 170), (120, 90, 75), 3, 4, 4, 3, 3, 3, 1),
    ("ring", 36, (160, 160), (80, 80, 0), 2, 2, 6, 20, 2, 1, 0),
    ("l_bracket", 64, (260, 200), (131, 97, 250), 4, 8, 2, 5, 2, 3, 0),
    ("cross", 36, (170, 130), (84, 66, 45), 2, 3, 5, 4, 1, 3, 0),
]


@pytest.mark.parametrize("case", range(len(C2F_SWEEP)))
def test_coarse_to_fine_sweep(ea, oracle, case):
    """search_levels across beam widths (topk 1..20), refinement radii 1-3,
    neighbourhoods 1/3/5, both polarities, 2-4 levels and grid steps that
    do and do not divide the level scale (a step of 3 at level 0 is a
    non-integer top-level step): Detector.detect == the oracle's
    coarse_to_fine, outcome and per-level trace."""
    tid, size, (W, H), (px, py, pt), L, st, dt, k, rr, nb, pol = C2F_SWEEP[case]
    img, tmpl = scene(ea, canvas_width=W, canvas_height=H, template_id=tid, template_size=size,
                      true_pose=(px, py, D(pt)), clutter_segments=12, clutter_seed=case,
                      noise_sigma=1.0, noise_seed=50 + case)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, W - 1, st, 0, H - 1, st, 0.0, D(360 - dt), D(dt)),
                          num_levels=L, score_params=ea.ScoreParams(nb, pol), topk=k,
                          refine_radius=rr, min_score=0.3)
    tp, wp = oracle.build_pyramid(tmpl, L), oracle.build_pyramid(img, L)
    want = oracle.coarse_to_fine(tp, wp, cfg)
    assert ea.Detector(tmpl, cfg).detect(img).key() == want.key()


def test_shared_context_interleaved_detects(ea, oracle):
    """Two detectors of different templates, image sizes, grids and
    neighbourhoods on ONE context, interleaved with batch calls: the
    context's caches (screening plane, exact-zero tiles, theta tables, tail
    and candidate buffers, refinement state) are keyed by what they depend
    on, so every result == the oracle."""
    ctx = ea.Context(0)
    specs = [
        (dict(canvas_width=240, canvas_height=180, template_id="l_bracket", template_size=56,
              true_pose=(118, 92, D(40)), clutter_segments=15, clutter_seed=3), 2, 3, 2),
        (dict(canvas_width=150, canvas_height=200, template_id="cross", template_size=40,
              true_pose=(70, 110, D(12)), clutter_segments=8, clutter_seed=4), 3, 5, 4),
    ]
    dets, imgs, wants = [], [], []
    for spec, L, nb, st in specs:
        img, tmpl = scene(ea, **spec)
        W, H = spec["canvas_width"], spec["canvas_height"]
        cfg = ea.SearchConfig(grid=ea.PoseGrid(0, W - 1, st, 0, H - 1, st, 0.0, D(356), D(4)),
                              num_levels=L, score_params=ea.ScoreParams(nb), topk=4,
                              min_score=0.3)
        dets.append(ea.Detector(tmpl, cfg, ctx))
        imgs.append(img)
        wants.append(oracle.coarse_to_fine(oracle.build_pyramid(tmpl, L),
                                           oracle.build_pyramid(img, L), cfg).key())
    for order in ((0, 1, 0, 1), (1, 1, 0, 0)):
        for i in order:
            assert dets[i].detect(imgs[i]).key() == wants[i], i
        for i in (1, 0):
            assert [o.key() for o in dets[i].detect_batch([imgs[i]] * 3)] == [wants[i]] * 3
    ctx.close()


def test_flat_scene_no_detection(ea, oracle):
    flat = np.full((96, 96), 180.0)
    tmpl = oracle.render_template("rectangle", 32)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(16, 80, 4, 16, 80, 4, 0.0, 0.0, 1.0), num_levels=2,
                          score_params=ea.ScoreParams(3))
    tp, wp = oracle.build_pyramid(tmpl, 2), oracle.build_pyramid(flat, 2)
    got = ea.coarse_to_fine(tp, wp, cfg)
    assert not got.found and got.score < cfg.min_score
    assert got.key() == oracle.coarse_to_fine(tp, wp, cfg).key()


def test_prepare_levels_errors(ea):
    flat = np.full((64, 64), 127.0)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 63, 4, 0, 63, 4, 0, 0, 1), num_levels=2)
    pyr = ea.build_pyramid(flat, 2)
    with pytest.raises(ea.EmptyModelError, match="level 0"):
        ea.prepare_levels(pyr, pyr, cfg)
    cfg.num_levels = 3
    with pytest.raises(ea.InvalidArgument, match="pyramids must provide 3 levels"):
        ea.prepare_levels(pyr, pyr, cfg)


def test_prepare_levels_models_and_fields(ea, oracle):
    img, tmpl = scene(ea, canvas_width=160, canvas_height=160, template_id="l_bracket",
                      template_size=48, true_pose=(80, 76, D(22)), clutter_segments=14,
                      clutter_seed=99)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 159, 2, 0, 159, 2, 0, D(10), D(5)), num_levels=2)
    tp, wp = oracle.build_pyramid(tmpl, 2), oracle.build_pyramid(img, 2)
    lv = ea.prepare_levels(tp, wp, cfg)
    models, fields = oracle.prepare_levels(tp, wp, cfg)
    for l in range(2):
        got = lv.model(l)
        assert np.array_equal(got.points, models[l].points)
        assert (got.centroid_x, got.centroid_y) == (models[l].centroid_x, models[l].centroid_y)
        for a, b in zip(lv.field(l), fields[l]):
            assert np.array_equal(a, b)


@pytest.mark.slow
def test_config1_detect_bit_exact(ea, oracle):
    """BASELINE configs[0]: 640x480, 128 px model, 1 deg over 360, 3 levels."""
    img, tmpl = scene(ea, canvas_width=640, canvas_height=480, template_id="l_bracket",
                      template_size=128, true_pose=(320, 240, D(30)), clutter_segments=40,
                      clutter_seed=7)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 639, 4, 0, 479, 4, 0.0, D(359), D(1)),
                          num_levels=3, score_params=ea.ScoreParams(3))
    tp, wp = oracle.build_pyramid(tmpl, 3), oracle.build_pyramid(img, 3)
    want = oracle.coarse_to_fine(tp, wp, cfg)
    got = ea.Detector(tmpl, cfg).detect(img)
    assert got.key() == want.key()
    assert got.found
    assert abs(got.pose.ux - 320) <= 2 and abs(got.pose.uy - 240) <= 2


@pytest.mark.slow
def test_config2_detect_bit_exact(ea, oracle):
    """BASELINE configs[1] (the bench workload): 1280x1024, 200 px model,
    0.5 deg over 360, 4 levels, occluder + illumination + noise."""
    import bench
    img, tmpl, cfg, truth = bench.make_inputs("cfg2")
    L = cfg.num_levels
    tp, wp = oracle.build_pyramid(tmpl, L), oracle.build_pyramid(img, L)
    want = oracle.coarse_to_fine(tp, wp, cfg)
    got = ea.Detector(tmpl, cfg).detect(img)
    assert got.key() == want.key()


def test_detect_batch_matches_single(ea, oracle):
    """Throughput-mode batch detect == per-image detect == oracle."""
    specs = [dict(canvas_width=160, canvas_height=128, template_id="l_bracket", template_size=48,
                  true_pose=(80 + 3 * i, 64 - 2 * i, D(20 + 35 * i)), clutter_segments=10 + i,
                  clutter_seed=i, noise_sigma=1.0 * (i % 2), noise_seed=7 + i) for i in range(5)]
    imgs, tmpl = [], None
    for kw in specs:
        img, t = scene(ea, **kw)
        imgs.append(img)
        tmpl = t
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 159, 2, 0, 127, 2, 0.0, D(355), D(5)),
                          num_levels=2, score_params=ea.ScoreParams(3))
    det = ea.Detector(tmpl, cfg)
    batch = det.detect_batch(imgs)
    tp = oracle.build_pyramid(tmpl, 2)
    for img, got in zip(imgs, batch):
        assert got.key() == det.detect(img).key()
        assert got.key() == oracle.coarse_to_fine(tp, oracle.build_pyramid(img, 2), cfg).key()
    # the same images staged in the library's pinned buffers (ea_host_alloc)
    pinned = []
    for img in imgs:
        buf = ea.host_array(img.shape)
        buf[...] = img
        pinned.append(buf)
    assert [o.key() for o in det.detect_batch(pinned)] == [o.key() for o in batch]
    assert det.detect(pinned[2]).key() == batch[2].key()


@pytest.mark.slow
def test_config3_detect_bit_exact(ea, oracle):
    """BASELINE configs[2]: 2592x1944 (5 MP), 256 px model, 0.25 deg full
    rotation, 5 levels (the theta-sharded config)."""
    import bench
    img, tmpl, cfg, truth = bench.make_inputs("cfg3")
    L = cfg.num_levels
    tp, wp = oracle.build_pyramid(tmpl, L), oracle.build_pyramid(img, L)
    want = oracle.coarse_to_fine(tp, wp, cfg)
    got = ea.Detector(tmpl, cfg).detect(img)
    assert got.key() == want.key()


@pytest.mark.slow
def test_config4_batch_bit_exact(ea, oracle):
    """BASELINE configs[3] (throughput mode): the first scenes of the cfg4
    batch through detect_batch == the oracle's coarse_to_fine, image by image."""
    import bench
    _, tmpl, cfg, _ = bench.make_inputs("cfg4")
    imgs = bench.batch_scenes("cfg4", 3)
    outs = ea.Detector(tmpl, cfg).detect_batch(imgs)
    L = cfg.num_levels
    tp = oracle.build_pyramid(tmpl, L)
    for img, got in zip(imgs, outs):
        assert got.key() == oracle.coarse_to_fine(tp, oracle.build_pyramid(img, L), cfg).key()


def test_detect_multi_matches_oracle(ea, oracle):
    """Multi-model detect on a multi-stamp scene whose top level (320x240)
    exceeds shared memory (region-tiled screening): each model's outcome ==
    its own Detector.detect == the oracle's coarse_to_fine."""
    stamps = [("l_bracket", 64, (150.0, 130.0, D(40))), ("cross", 96, (460.0, 140.0, D(15))),
              ("ring", 80, (170.0, 350.0, 0.0)), ("rectangle", 72, (470.0, 340.0, D(200)))]
    spec = ea.SceneSpec(640, 480, "rectangle", 0, (0, 0, 0), 60, 5, None, (1.1, 4.0, 1.0), 1.5, 9)
    img = ea.compose_multi(spec, stamps)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 639, 2, 0, 479, 2, 0.0, D(350), D(10)),
                          num_levels=2, score_params=ea.ScoreParams(3), topk=3)
    tmpls = [ea.render_template(t, s) for t, s, _ in stamps]
    dets = [ea.Detector(t, cfg) for t in tmpls]
    outs = ea.detect_multi(dets, img)
    wp = oracle.build_pyramid(img, 2)
    for t, d, got in zip(tmpls, dets, outs):
        want = oracle.coarse_to_fine(oracle.build_pyramid(t, 2), wp, cfg)
        assert got.key() == want.key()
        assert got.key() == d.detect(img).key()
    assert ea.default_context().stats()["screen_path"] == 3


@pytest.mark.slow
def test_config5_multi_detect_bit_exact(ea, oracle):
    """BASELINE configs[4]: 2592x1944 cluttered multi-stamp scene, 8 models
    (64-400 px), 0.5 deg, 4 levels: detect_multi == oracle, model by model."""
    import bench
    img, tmpls, cfg, _ = bench.make_multi_inputs("cfg5")
    L = cfg.num_levels
    dets = [ea.Detector(t, cfg) for t in tmpls]
    outs = ea.detect_multi(dets, img)
    wp = oracle.build_pyramid(img, L)
    # Parity only: under 400 clutter segments the reference's top-k beam
    # (5 seeds, no spatial suppression) locks onto clutter for several of the
    # small/symmetric models, and so must we.
    for t, got in zip(tmpls, outs):
        want = oracle.coarse_to_fine(oracle.build_pyramid(t, L), wp, cfg)
        assert got.key() == want.key()


@pytest.mark.parametrize("G", [1, 3, 8])
def test_sharded_detect_flow(ea, oracle, G):
    """The multi-GPU detect on one device: theta-slab top-level searches
    (search_top_slab, one per rank), the `better` merge (what gather_topk
    does over NCCL), then refine from the merged seeds == detect == oracle."""
    img, tmpl = scene(ea, canvas_width=200, canvas_height=160, template_id="l_bracket",
                      template_size=56, true_pose=(96, 84, D(63)), clutter_segments=25,
                      clutter_seed=4, noise_sigma=1.0, noise_seed=2)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 199, 4, 0, 159, 4, 0.0, D(357), D(3)),
                          num_levels=3, score_params=ea.ScoreParams(3), topk=4)
    det = ea.Detector(tmpl, cfg)
    want = det.detect(img)
    nt = ea.grid_counts(ea.PoseGrid(0, 49.75, 1, 0, 39.75, 1, 0.0, D(357), D(3)))[2]
    seeds = []
    for g in range(G):
        seeds += ea.search_top_slab(det.levels, cfg, nt * g // G, nt * (g + 1) // G)
    got = ea.refine(det.levels, cfg, ea.merge_topk(seeds, cfg.topk))
    assert got.key() == want.key()
    tp, wp = oracle.build_pyramid(tmpl, 3), oracle.build_pyramid(img, 3)
    assert got.key() == oracle.coarse_to_fine(tp, wp, cfg).key()


# ---- template side on the device ----------------------------------------
def model_key(m):
    return (np.asarray(m.points).tobytes(), m.centroid_x, m.centroid_y)


@pytest.mark.parametrize("shape", ["rectangle", "ring", "l_bracket", "cross"])
@pytest.mark.parametrize("size", [16, 33, 64, 200, 400])
def test_device_edge_model_templates(ea, oracle, shape, size):
    img = oracle.render_template(shape, size)
    f = oracle.compute_gradients(img)
    got = ea.extract_edge_model_device(f)
    want = oracle.extract_edge_model(f, oracle.default_thresholds(f), 0)
    assert model_key(got) == model_key(want)


@pytest.mark.parametrize("seed", range(4))
def test_device_edge_model_random_fields(ea, oracle, seed):
    rng = np.random.default_rng(500 + seed)
    f = oracle.compute_gradients(rand_image(rng, 57 + seed, 43, real=seed % 2 == 1))
    for th in (None, (0.0, 0.0), (10.0, 10.0), (5.0, 300.0)):
        want_th = oracle.default_thresholds(f) if th is None else th
        got = ea.extract_edge_model_device(f, th)
        want = oracle.extract_edge_model(f, want_th, 0)
        assert model_key(got) == model_key(want)


def test_device_edge_model_boundary_bins(ea, oracle):
    """Gradients exactly on the 22.5/67.5/112.5/157.5 degree bin boundaries
    (in fp64) go to the host's atan2 and must bin like the reference."""
    rng = np.random.default_rng(9)
    h, w = 24, 30
    gx = rng.normal(size=(h, w)) * 20
    gy = rng.normal(size=(h, w)) * 20
    t = 0.41421356237309503
    dirs = [(1.0, t), (t, 1.0), (-t, 1.0), (-1.0, t), (1.0, -t), (-t, -1.0), (t, -1.0)]
    for k in range(200):
        y, x = 1 + rng.integers(0, h - 2), 1 + rng.integers(0, w - 2)
        s = float(rng.integers(1, 50))
        gx[y, x], gy[y, x] = dirs[k % len(dirs)][0] * s, dirs[k % len(dirs)][1] * s
    gx[0, :] = gx[-1, :] = gx[:, 0] = gx[:, -1] = 0.0
    gy[0, :] = gy[-1, :] = gy[:, 0] = gy[:, -1] = 0.0
    mag = np.sqrt(gx * gx + gy * gy)
    f = (gx, gy, mag)
    for th in (None, (1.0, 30.0)):
        want_th = oracle.default_thresholds(f) if th is None else th
        assert model_key(ea.extract_edge_model_device(f, th)) == \
            model_key(oracle.extract_edge_model(f, want_th, 0))


def test_device_edge_model_errors(ea):
    z = np.zeros((9, 9))
    with pytest.raises(ea.EmptyModelError, match="empty model"):
        ea.extract_edge_model_device((z, z, z))
    f = ea.compute_gradients(np.arange(100.0).reshape(10, 10) ** 2)
    with pytest.raises(ea.InvalidArgument, match="0 <= low <= high"):
        ea.extract_edge_model_device(f, (5.0, 1.0))


def test_async_slab_rows_and_device_merge(ea, oracle):
    """Device-resident slab search rows == ea_search_top_slab; the device
    merge of all slabs' rows == merge_topk == the full search."""
    import torch
    img, tmpl = scene(ea, canvas_width=200, canvas_height=160, template_id="l_bracket",
                      template_size=56, true_pose=(96, 84, D(63)), clutter_segments=25,
                      clutter_seed=4)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 199, 4, 0, 159, 4, 0.0, D(357), D(3)),
                          num_levels=3, score_params=ea.ScoreParams(3), topk=6)
    det = ea.Detector(tmpl, cfg)
    det.levels.set_image(img)
    ctx = det.ctx
    nt = 120
    G, k = 5, cfg.topk
    rows = torch.empty((G * k, 5), dtype=torch.float64, device="cuda")
    seeds = []
    for g in range(G):
        a, b = nt * g // G, nt * (g + 1) // G
        ea.search_top_slab_async(det.levels, cfg, a, b, rows[g * k:(g + 1) * k].data_ptr())
        seeds.append(ea.search_top_slab(det.levels, cfg, a, b))
    merged = torch.empty((k, 5), dtype=torch.float64, device="cuda")
    ea.merge_rows_async(ctx, rows.data_ptr(), G * k, k, merged.data_ptr())
    overflowed, _ = ea.async_status(ctx)
    assert not overflowed
    from paper_2112_05576_b200 import parallel
    got = rows.cpu().numpy()
    for g in range(G):
        assert parallel.unpack(got[g * k:(g + 1) * k]) == [s for s in seeds[g]] or \
            [(s.score, s.grid_index, s.pose.astuple()) for s in parallel.unpack(got[g * k:(g + 1) * k])] == \
            [(s.score, s.grid_index, s.pose.astuple()) for s in seeds[g]]
    want = ea.merge_topk([s for part in seeds for s in part], k)
    full = ea.search_top_slab(det.levels, cfg, 0, nt)
    key = lambda lst: [(s.score, int(s.grid_index), s.pose.astuple()) for s in lst]
    assert key(parallel.unpack(merged.cpu().numpy())) == key(want) == key(full)


def test_gather_rows_device_nccl_single_rank(ea, oracle):
    """The bench's N-GPU exchange on one rank: NCCL all-gather of the device
    rows + device merge == the local rows (world size 1)."""
    import os
    import socket

    import torch
    import torch.distributed as dist
    from paper_2112_05576_b200 import parallel

    img, tmpl = scene(ea, canvas_width=160, canvas_height=128, template_id="l_bracket",
                      template_size=48, true_pose=(80, 64, D(20)), clutter_segments=10,
                      clutter_seed=3)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 159, 2, 0, 127, 2, 0.0, D(355), D(5)),
                          num_levels=2, score_params=ea.ScoreParams(3), topk=5)
    det = ea.Detector(tmpl, cfg)
    det.levels.set_image(img)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        parallel.init_comm(det.ctx)  # the library's own NCCL communicator (id over torch)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            det.ctx.set_stream(stream.cuda_stream)
            rows = torch.empty((5, 5), dtype=torch.float64, device="cuda")
            ea.search_top_slab_async(det.levels, cfg, 0, 72, rows.data_ptr())
            merged = parallel.gather_rows_device(rows, 5, det.ctx)
            stream.synchronize()
        want = ea.search_top_slab(det.levels, cfg, 0, 72)
        key = lambda lst: [(s.score, int(s.grid_index), s.pose.astuple()) for s in lst]
        assert key(parallel.unpack(merged.cpu().numpy())) == key(want)
    finally:
        dist.destroy_process_group()
        det.ctx.set_stream(None)
        det.ctx.comm_destroy()


def test_plane_cache_follows_field_and_params(ea, oracle):
    """The screening plane is cached per (field, version, eps, geometry): a
    search must see a new image after set_image (same field objects), another
    field, another eps, and a screen_map (which leaves the histogram dirty)
    between searches -- each result equal to the oracle's."""
    rng = np.random.default_rng(2024)
    m = rand_model(oracle, rng, 14)
    imgs = [rand_image(rng, 48, 40) for _ in range(3)]
    fields = [oracle.compute_gradients(im) for im in imgs]
    dfields = [ea.DeviceField.upload(f) for f in fields]
    grid = ea.PoseGrid(0, 47, 1, 0, 39, 1, 0.0, D(350), D(10))
    dm = ea.DeviceModel(m)
    seq = [(0, 1e-9), (1, 1e-9), (0, 1e-9), (0, 5.0), (2, 1e-9), ("map", 1e-9), (2, 1e-9),
           (1, 5.0), (1, 5.0)]
    for which, eps in seq:
        params = ea.ScoreParams(3, 0, eps)
        if which == "map":
            ea.screen_map(dm, dfields[2], grid, params)
            continue
        got = ea.search_topk(dm, dfields[which], grid, params, k=5)
        want = oracle.search_topk(m.points, fields[which], grid, params, 5)
        assert keys(got) == keys(want), (which, eps)
    # same levels object, new images (the fields are rewritten in place)
    tmpl = imgs[0][4:36, 8:40]
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 47, 2, 0, 39, 2, 0.0, D(350), D(10)),
                          num_levels=2, score_params=ea.ScoreParams(3))
    det = ea.Detector(tmpl, cfg)
    tp = oracle.build_pyramid(tmpl, 2)
    for im in imgs + imgs[:1]:
        got = det.detect(im)
        assert got.key() == oracle.coarse_to_fine(tp, oracle.build_pyramid(im, 2), cfg).key()


@pytest.mark.parametrize("case", [0, 3, len(SEARCH_CASES) - 1])
def test_unfused_finish_path_matches(ea, oracle, monkeypatch, case):
    """EAB_NO_FUSED_FINISH=1 (read at context creation) runs the separate
    compact / rescore / select kernels instead of the cooperative finish
    kernel: both must give the oracle's top k, on contexts used back to back."""
    size, w, h, g, nb, pol = SEARCH_CASES[case]
    rng = np.random.default_rng(300 + case)
    m = rand_model(oracle, rng, size)
    f = oracle.compute_gradients(rand_image(rng, w, h))
    grid = ea.PoseGrid(*g)
    params = ea.ScoreParams(nb, pol)
    want = keys(oracle.search_topk(m.points, f, grid, params, 7))
    monkeypatch.setenv("EAB_NO_FUSED_FINISH", "1")
    ctx_sep = ea.Context(0)
    monkeypatch.delenv("EAB_NO_FUSED_FINISH")
    ctx_fused = ea.Context(0)
    for ctx in (ctx_sep, ctx_fused, ctx_sep):
        assert keys(ea.search_topk(m, f, grid, params, k=7, ctx=ctx)) == want
    ctx_sep.close()
    ctx_fused.close()


@pytest.mark.parametrize("case", [0, 1, 2, 3, 4, 5, len(SEARCH_CASES) - 1])
def test_screen_threshold_modes_match(ea, oracle, monkeypatch, case):
    """Three ways to the band threshold, all equal to the oracle for every k,
    on contexts used back to back (shared model caches, plane cache):
    top-list mode (default for k <= 8 on the smem lattice kernel: no
    histogram, threshold from the k-th largest tile maximum), the histogram
    (EAB_NO_TOPLIST=1, and always for k > 8), and the screen with the finish
    inside its cooperative launch (EAB_FUSED_SCREEN=1)."""
    size, w, h, g, nb, pol = SEARCH_CASES[case]
    rng = np.random.default_rng(900 + case)
    m = rand_model(oracle, rng, size)
    f = oracle.compute_gradients(rand_image(rng, w, h))
    grid = ea.PoseGrid(*g)
    params = ea.ScoreParams(nb, pol)
    monkeypatch.setenv("EAB_NO_TOPLIST", "1")
    ctx_hist = ea.Context(0)
    monkeypatch.delenv("EAB_NO_TOPLIST")
    monkeypatch.setenv("EAB_FUSED_SCREEN", "1")
    ctx_fused = ea.Context(0)
    monkeypatch.delenv("EAB_FUSED_SCREEN")
    ctx_top = ea.Context(0)
    for k in (1, 2, 5, 8, 9):
        want = keys(oracle.search_topk(m.points, f, grid, params, k))
        for ctx in (ctx_top, ctx_hist, ctx_fused, ctx_top, ctx_fused):
            assert keys(ea.search_topk(m, f, grid, params, k=k, ctx=ctx)) == want, (k, ctx)
    for c in (ctx_hist, ctx_fused, ctx_top):
        c.close()


@pytest.mark.parametrize("tid,size", [("cross", 40), ("rectangle", 48), ("ring", 36)])
def test_toplist_clustered_peak(ea, oracle, monkeypatch, tid, size):
    """A lone clean object on a blank canvas: the k best poses all sit in the
    peak's warp tile (adjacent translations and thetas).  The top lists then
    hold that tile's lane maxima -- distinct poses, so the band threshold
    stays <= T_f -- and the map floor rises after the first tile.  Default
    (top lists) and histogram paths == the oracle for k up to 8 and 9."""
    img, tmpl = scene(ea, canvas_width=160, canvas_height=120, template_id=tid,
                      template_size=size, true_pose=(80, 60, D(25)), clutter_segments=0,
                      clutter_seed=1, noise_sigma=0.0, noise_seed=1)
    m = oracle.prepare_model(tmpl)
    f = oracle.compute_gradients(img)
    grid = ea.PoseGrid(0, 159, 1, 0, 119, 1, 0.0, D(359), D(1))
    params = ea.ScoreParams(3)
    monkeypatch.setenv("EAB_NO_TOPLIST", "1")
    ctx_hist = ea.Context(0)
    monkeypatch.delenv("EAB_NO_TOPLIST")
    ctx_top = ea.Context(0)
    for k in (1, 5, 8, 9):
        want = keys(oracle.search_topk(m.points, f, grid, params, k))
        for ctx in (ctx_top, ctx_hist):
            assert keys(ea.search_topk(m, f, grid, params, k=k, ctx=ctx)) == want, (k, ctx)
    ctx_hist.close()
    ctx_top.close()


def test_fused_screen_ties_and_tiny_grids(ea, oracle, monkeypatch):
    """Top-list and fused path edge cases: a flat field (every pose ties at 0: the k-th
    largest is 0 and every pose is a candidate), grids with fewer poses than
    k, and one-theta grids."""
    rng = np.random.default_rng(77)
    m = rand_model(oracle, rng, 10)
    flat = oracle.compute_gradients(np.full((24, 20), 42.0))
    f = oracle.compute_gradients(rand_image(rng, 24, 20))
    params = ea.ScoreParams(3)
    monkeypatch.setenv("EAB_FUSED_SCREEN", "1")
    ctx_fused = ea.Context(0)
    monkeypatch.delenv("EAB_FUSED_SCREEN")
    for field, ctx in ((flat, None), (f, None), (flat, ctx_fused), (f, ctx_fused)):
        for g in ((0, 19, 1, 0, 23, 1, 0.0, D(20), D(10)), (3, 4, 1, 5, 5, 1, 0.0, 0.0, 1.0),
                  (0, 1, 1, 0, 1, 1, 0.0, D(10), D(10)), (0, 19, 1, 0, 23, 1, D(7), D(7), 1.0)):
            grid = ea.PoseGrid(*g)
            for k in (1, 3, 8):
                want = keys(oracle.search_topk(m.points, field, grid, params, k))
                assert keys(ea.search_topk(m, field, grid, params, k=k, ctx=ctx)) == want, (g, k)
    ctx_fused.close()


@pytest.mark.parametrize("w,h,L", [(160, 160, 1), (333, 257, 4), (162, 121, 2), (648, 486, 5),
                                   (517, 389, 6), (97, 64, 3)])
def test_fused_pyramid_fields_bit_exact(ea, oracle, monkeypatch, w, h, L):
    """set_image builds every level's image and gradient field in one kernel
    (pyramid_fields_kernel, odd sizes, 1-6 levels); EAB_NO_FUSED_PYRAMID=1
    runs the per-level downsample + Sobel kernels.  Both equal the oracle."""
    rng = np.random.default_rng(w * 7 + h * 3 + L)
    tmpl = rand_image(rng, 8 << (L - 1), 8 << (L - 1), real=True)
    img = rand_image(rng, w, h, real=True)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, w - 1, 1 << (L - 1), 0, h - 1, 1 << (L - 1),
                                           0.0, D(90), D(45)), num_levels=L)
    tp = oracle.build_pyramid(tmpl, L)
    wp = oracle.build_pyramid(img, L)
    want = [oracle.compute_gradients(level) for level in wp]
    lv = ea.prepare_levels(tp, wp, cfg)
    for fused in (True, False):
        if not fused:
            monkeypatch.setenv("EAB_NO_FUSED_PYRAMID", "1")
        lv.set_image(img)
        for l in range(L):
            for a, b in zip(lv.field(l), want[l]):
                assert np.array_equal(a, b), (fused, l)
    monkeypatch.delenv("EAB_NO_FUSED_PYRAMID", raising=False)


# ---- integer steps > 1 on the lattice kernels (unit lattice, strided emit) --------------
STRIDE_CASES = [
    # (model size, field w, h, grid, nb, polarity)
    (12, 64, 48, (0, 63, 2, 0, 47, 2, 0.0, D(350), D(10)), 3, 0),
    (12, 64, 48, (1, 62, 3, 2, 47, 3, 0.0, D(350), D(10)), 3, 0),
    (10, 60, 50, (-7, 66, 2, -5, 52, 3, 0.1, D(300), D(25)), 3, 0),   # off-image overhang
    (14, 64, 64, (0, 63, 3, 0, 63, 1, 0.0, D(357), D(3)), 1, 0),
    (14, 64, 64, (3, 60, 4, 3, 60, 4, 0.0, D(350), D(10)), 5, 1),
    (12, 300, 260, (0, 299, 3, 0, 259, 3, 0.0, D(345), D(15)), 3, 0),  # region-tiled plane
]


@pytest.mark.parametrize("case", range(len(STRIDE_CASES)))
def test_strided_lattice_bit_exact(ea, oracle, case):
    """Integer steps > 1 (the paper's 3 px / 3 px grid) run the lattice
    kernels over the unit lattice covering the grid and emit only the grid's
    poses: same top k as the oracle for k in and beyond the top-list range."""
    size, w, h, g, nb, pol = STRIDE_CASES[case]
    rng = np.random.default_rng(700 + case)
    m = rand_model(oracle, rng, size)
    f = oracle.compute_gradients(rand_image(rng, w, h, real=case % 2 == 1))
    grid = ea.PoseGrid(*g)
    params = ea.ScoreParams(nb, pol)
    for k in (1, 5, 11):
        got = ea.search_topk(m, f, grid, params, k=k)
        assert ea.default_context().stats()["screen_path"] in (1, 3)  # a lattice kernel
        assert keys(got) == keys(oracle.search_topk(m.points, f, grid, params, k)), k


@pytest.mark.slow
def test_paper_geometry_detect_bit_exact(ea, oracle):
    """The paper's own experiment geometry: an
    812 x 617 search image, steps of 3 px / 3 px / 3 deg over the full
    rotation, searched at level 0 -- the strided lattice path; detect ==
    the oracle's coarse_to_fine bit for bit."""
    img, tmpl = scene(ea, canvas_width=812, canvas_height=617, template_id="l_bracket",
                      template_size=96, true_pose=(400, 300, D(42)), clutter_segments=40,
                      clutter_seed=21, noise_sigma=1.5, noise_seed=4)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(0, 811, 3, 0, 616, 3, 0.0, D(357), D(3)),
                          num_levels=1, score_params=ea.ScoreParams(3), topk=5)
    got = ea.Detector(tmpl, cfg).detect(img)
    assert ea.default_context().stats()["screen_path"] == 3
    want = oracle.coarse_to_fine(oracle.build_pyramid(tmpl, 1), oracle.build_pyramid(img, 1), cfg,
                                 threads=16)
    assert got.key() == want.key()
    assert got.found
