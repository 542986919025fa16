"""The reference's own test cases (proj/tests/test_*.cpp), restated.

They run on CPU against the C oracle; the `product_host` variants run the
product's host-side C-ABI (pose geometry, template-side extraction, merge,
synth) which needs no GPU.  Device-side equivalents live in
tests/test_gpu_parity.py.
"""
import math

import numpy as np
import pytest

import paper_2112_05576_b200 as ea
from paper_2112_05576_b200 import abi

D = abi.deg_to_rad


# ---- test_pose.cpp ------------------------------------------------------------------------
@pytest.fixture(params=["oracle", "product_host"])
def geo(request, oracle):
    if request.param == "oracle":
        return (lambda g: tuple(oracle.grid_counts(g)),
                lambda g, i: tuple(oracle.pose_at(g, i)))
    return (lambda g: tuple(ea.grid_counts(g)), lambda g, i: ea.pose_at(g, i).astuple())


def test_grid_size_matches_count_formula(geo):  # test_pose.cpp:79-93
    counts, _ = geo
    assert counts(ea.PoseGrid(0, 812, 3, 0, 615, 3, 0, D(87), D(3))) == (271, 206, 30)
    assert math.prod(counts(ea.PoseGrid(0, 812, 3, 0, 615, 3, 0, D(87), D(3)))) == 1674780
    assert math.prod(counts(ea.PoseGrid(4, 4, 1, 5, 5, 1, 0.2, 0.2, 0.1))) == 1
    assert math.prod(counts(ea.PoseGrid(0, 4, 2, 1, 1, 1, 0, 0, 1))) == 3


def test_grid_validation(geo):  # test_pose.cpp:95-100
    counts, _ = geo
    with pytest.raises(ea.InvalidArgument):
        counts(ea.PoseGrid(0, 1, 0.0, 0, 1, 1, 0, 1, 1))
    with pytest.raises(ea.InvalidArgument):
        counts(ea.PoseGrid(2, 1, 1, 0, 1, 1, 0, 1, 1))
    with pytest.raises(ea.InvalidArgument, match="non-finite"):
        counts(ea.PoseGrid(0, float("inf"), 1, 0, 1, 1, 0, 1, 1))


def test_pose_at_theta_major(geo):  # test_pose.cpp:102-125
    counts, at = geo
    g = ea.PoseGrid(10, 14, 2, 20, 26, 3, 0.5, 0.9, 0.2)
    assert counts(g) == (3, 3, 3)
    assert at(g, 0) == (10.0, 20.0, 0.5)
    assert at(g, 3) == (10.0, 23.0, 0.5)
    last = at(g, 26)
    assert last[:2] == (14.0, 26.0) and last[2] == pytest.approx(0.9)
    with pytest.raises(ea.BoundsError, match="out of range"):
        at(g, 27)


def test_pose_at_bijection(geo):  # test_pose.cpp:127-136
    counts, at = geo
    g = ea.PoseGrid(-3, 3, 1.5, 0, 4, 2, 0, D(30), D(15))
    total = math.prod(counts(g))
    assert len({at(g, i) for i in range(total)}) == total


# ---- test_image.cpp -------------------------------------------------------------------------
def test_box_mean_kat(oracle):  # test_image.cpp:125-132
    out = oracle.downsample(np.array([[0.0, 0.0], [4.0, 4.0]]))
    assert out.shape == (1, 1) and out[0, 0] == 2.0


def test_downsample_preserves_constants(oracle):  # test_image.cpp:134-149
    rng = np.random.default_rng(11)
    for _ in range(10):
        v = rng.uniform(-40, 300)
        assert (oracle.downsample(np.full((4, 6), v)) == v).all()
    assert (oracle.downsample(np.full((4, 4), 9.0)) == 9.0).all()


def test_downsample_odd_and_small(oracle):  # test_image.cpp:151-161
    assert oracle.downsample(np.ones((5, 5))).shape == (2, 2)
    with pytest.raises(ea.SizeError):
        oracle.downsample(np.zeros((5, 1)))


def test_pyramid_dims_and_levels(oracle):  # test_image.cpp:163-202
    img = np.arange(130.0).reshape(13, 10)
    assert np.array_equal(oracle.build_pyramid(img, 1)[0], img)
    pyr = oracle.build_pyramid(np.zeros((617, 812)), 3)
    assert [p.shape for p in pyr] == [(617, 812), (308, 406), (154, 203)]
    with pytest.raises(ea.SizeError, match="2"):
        oracle.build_pyramid(np.zeros((16, 16)), 4)
    assert oracle.max_pyramid_levels(16, 16) == 2 == ea.max_pyramid_levels(16, 16)
    assert len(oracle.build_pyramid(np.zeros((16, 16)), 2)) == 2


# ---- test_edge_model.cpp ----------------------------------------------------------------------
def vertical_step(w, h, first, lo, hi):
    img = np.full((h, w), lo)
    img[:, first:] = hi
    return img


def test_sobel_kats(oracle):  # test_edge_model.cpp:50-92
    f = oracle.compute_gradients(np.full((7, 9), 123.25))
    assert not any(a.any() for a in f)
    with pytest.raises(ea.SizeError):
        oracle.compute_gradients(np.zeros((8, 2)))
    gx, gy, mag = oracle.compute_gradients(vertical_step(9, 7, 4, 0.0, 8.0))
    assert (gx[1:6, 3] == 32).all() and (gx[1:6, 4] == 32).all()
    assert (gy[1:6, 3:5] == 0).all() and (gx[1:6, 2] == 0).all() and (gx[1:6, 5] == 0).all()
    assert (mag[1:6, 3] == 32).all()
    img = np.zeros((9, 7))
    img[4:, :] = 8.0
    gx, gy, mag = oracle.compute_gradients(img)
    assert (gy[3, 1:6] == 32).all() and (gy[4, 1:6] == 32).all() and (gx[3, 1:6] == 0).all()


def test_border_ring_and_magnitude(oracle):  # test_edge_model.cpp:94-111
    rng = np.random.default_rng(3)
    gx, gy, mag = oracle.compute_gradients(rng.integers(0, 256, (11, 14)).astype(float))
    assert not mag[0].any() and not mag[-1].any() and not mag[:, 0].any() and not mag[:, -1].any()
    assert np.allclose(mag, np.sqrt(gx * gx + gy * gy), rtol=1e-9, atol=0)


def test_dyadic_gain_equivariance(oracle):  # test_edge_model.cpp:113-130
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (12, 16)).astype(float)
    base = oracle.compute_gradients(img)
    for a in (0.25, 0.5, 2.0, 4.0):
        for b in (-30.0, 0.0, 50.0):
            f = oracle.compute_gradients(a * img + b)
            assert np.array_equal(f[0], a * base[0]) and np.array_equal(f[1], a * base[1])


@pytest.fixture(params=["oracle", "product_host"])
def extract(request, oracle):
    if request.param == "oracle":
        return oracle.extract_edge_model, oracle.default_thresholds
    return ea.extract_edge_model, ea.default_thresholds


def test_flat_field_empty_model(oracle, extract):  # test_edge_model.cpp:132-140
    ext, _ = extract
    f = oracle.compute_gradients(np.full((9, 9), 55.0))
    with pytest.raises(ea.EmptyModelError) as e:
        ext(f, (0.0, 0.0), 0)
    assert e.value.max_magnitude == 0.0


def test_ideal_step_single_column(oracle, extract):  # test_edge_model.cpp:142-157
    ext, _ = extract
    m = ext(oracle.compute_gradients(vertical_step(11, 9, 5, 0.0, 8.0)), (1.0, 10.0), 0)
    cols = {round(p[0] + m.centroid_x) for p in m.points}
    assert len(cols) == 1
    assert np.all(np.abs(np.abs(m.points[:, 2]) - 1.0) < 1e-12)
    assert np.all(np.abs(m.points[:, 3]) < 1e-12)


def test_thresholds_subset_and_monotone(oracle, extract):  # test_edge_model.cpp:159-239
    ext, dth = extract
    rng = np.random.default_rng(8)
    f = oracle.compute_gradients(rng.integers(0, 256, (15, 15)).astype(float))
    px = lambda m: {(round(p[0] + m.centroid_x), round(p[1] + m.centroid_y)) for p in m.points}
    allm, some = ext(f, (0.0, 0.0), 0), ext(f, (2.0, 40.0), 0)
    assert px(some) <= px(allm)
    rng = np.random.default_rng(10)
    f = oracle.compute_gradients(rng.integers(0, 256, (18, 18)).astype(float))
    prev = 1e9
    for high in (0.0, 20.0, 60.0, 120.0):
        try:
            n = len(ext(f, (0.5 * high, high), 0).points)
        except ea.EmptyModelError:
            n = 0
        assert n <= prev
        prev = n
    rng = np.random.default_rng(12)
    f = oracle.compute_gradients(rng.integers(0, 256, (12, 12)).astype(float))
    lo, hi = dth(f)
    assert hi == pytest.approx(0.3 * f[2].max()) and lo == pytest.approx(0.15 * f[2].max())
    with pytest.raises(ea.InvalidArgument, match="0 <= low <= high"):
        ext(f, (5.0, 1.0), 0)


def test_model_invariants(oracle, extract):  # test_edge_model.cpp:208-228
    ext, _ = extract
    rng = np.random.default_rng(9)
    for _ in range(8):
        m = ext(oracle.compute_gradients(rng.integers(0, 256, (17, 20)).astype(float)),
                (0.0, 0.0), 2)
        assert np.all(np.abs(np.hypot(m.points[:, 2], m.points[:, 3]) - 1) <= 1e-9)
        assert np.all(m.points[:, 4] > 0)
        assert abs(m.points[:, 0].mean()) <= 1e-6 and abs(m.points[:, 1].mean()) <= 1e-6


# ---- test_similarity.cpp ------------------------------------------------------------------------
def field_with(w, h, sets):
    gx, gy = np.zeros((h, w)), np.zeros((h, w))
    for x, y, a, b in sets:
        gx[y, x], gy[y, x] = a, b
    return gx, gy, np.sqrt(gx * gx + gy * gy)


def test_point_vote_kats(oracle):  # test_similarity.cpp:45-81
    P = ea.ScoreParams
    assert oracle.point_vote(1, 0, field_with(7, 7, [(3, 3, 5, 0)]), 3, 3, P(3)) == \
        pytest.approx(1.0, abs=1e-12)
    assert oracle.point_vote(1, 0, field_with(7, 7, []), 3, 3, P(3)) == 0.0
    f = field_with(7, 7, [(3, 3, -5, 0), (4, 3, 1e-4, 0)])
    assert oracle.point_vote(1, 0, f, 3, 3, P(3)) == pytest.approx(1.0, abs=1e-12)
    assert oracle.point_vote(1, 0, f, 3, 3, P(1)) == pytest.approx(-1.0, abs=1e-12)
    z = field_with(5, 5, [])
    assert oracle.point_vote(0, 1, z, 40, 40, P(3)) == 0.0
    assert oracle.point_vote(0, 1, z, -9, 2, P(3)) == 0.0
    assert oracle.point_vote(1, 0, field_with(5, 5, [(2, 2, -7, 0)]), 2, 2,
                             P(1, abi.POLARITY_IGNORE)) == pytest.approx(1.0)


@pytest.mark.parametrize("tid", ["rectangle", "ring", "l_bracket", "cross"])
def test_self_match(oracle, tid):  # test_similarity.cpp:83-95
    tmpl = oracle.render_template(tid, 48)
    f = oracle.compute_gradients(tmpl)
    m = oracle.extract_edge_model(f, oracle.default_thresholds(f), 0)
    v, n = oracle.pose_score(m.points, (m.centroid_x, m.centroid_y, 0.0), f, ea.ScoreParams(1))
    assert v == pytest.approx(1.0, abs=1e-6) and n == len(m.points)


def test_zero_field_and_out_of_bounds(oracle):  # test_similarity.cpp:97-114
    m = oracle.prepare_model(oracle.render_template("rectangle", 32))
    z = np.zeros((64, 64))
    assert oracle.pose_score(m.points, (32, 32, 0), (z, z, z), ea.ScoreParams(3)) == \
        (0.0, len(m.points))
    rng = np.random.default_rng(31)
    f = oracle.compute_gradients(rng.integers(0, 256, (48, 48)).astype(float))
    assert oracle.pose_score(m.points, (500, 500, 0.3), f, ea.ScoreParams(3)) == (0.0, 0)


def test_score_bounds_and_monotone_neighbourhood(oracle):  # test_similarity.cpp:116-149
    rng = np.random.default_rng(37)
    m = oracle.prepare_model(oracle.render_template("cross", 32))
    f = oracle.compute_gradients(rng.integers(0, 256, (48, 48)).astype(float))
    for trial in range(100):
        pose = (rng.uniform(-10, 58), rng.uniform(-10, 58), rng.uniform(-3.2, 3.2))
        s = oracle.pose_score(m.points, pose, f, ea.ScoreParams(1 + 2 * (trial % 2)))[0]
        a = oracle.pose_score(m.points, pose, f, ea.ScoreParams(3, abi.POLARITY_IGNORE))[0]
        assert -1 - 1e-9 <= s <= 1 + 1e-9 and 0 <= a <= 1 + 1e-9
        n1, n3, n5 = (oracle.pose_score(m.points, pose, f, ea.ScoreParams(k))[0] for k in (1, 3, 5))
        assert n3 >= n1 and n5 >= n3


def test_affine_luminance_invariance(oracle):  # test_similarity.cpp:151-180
    rng = np.random.default_rng(43)
    img = rng.integers(0, 256, (48, 48)).astype(float)
    base = oracle.compute_gradients(img)
    m = oracle.prepare_model(oracle.render_template("rectangle", 32))
    poses = [(rng.uniform(6, 42), rng.uniform(6, 42), D(rng.uniform(6, 42))) for _ in range(40)]
    for a in (0.25, 1.7, 4.0):
        for b in (-30.0, 0.0, 50.0):
            f = oracle.compute_gradients(a * img + b)
            for pose in poses:
                assert abs(oracle.pose_score(m.points, pose, base, ea.ScoreParams(3))[0] -
                           oracle.pose_score(m.points, pose, f, ea.ScoreParams(3))[0]) <= 1e-9


# ---- test_search.cpp -----------------------------------------------------------------------------
def rand_model(oracle, rng, size):
    f = oracle.compute_gradients(rng.integers(0, 256, (size, size)).astype(float))
    return oracle.extract_edge_model(f, (0.0, 0.0), 0)


def test_single_pose_grid(oracle):  # test_search.cpp:40-53
    rng = np.random.default_rng(53)
    m = rand_model(oracle, rng, 10)
    f = oracle.compute_gradients(rng.integers(0, 256, (32, 32)).astype(float))
    g = ea.PoseGrid(16, 16, 1, 12, 12, 1, 0.2, 0.2, 0.1)
    d = oracle.exhaustive_search(m.points, f, g, ea.ScoreParams(3))
    assert d.grid_index == 0 and d.pose.astuple() == (16.0, 12.0, 0.2)
    assert d.score == oracle.pose_score(m.points, d.pose.astuple(), f, ea.ScoreParams(3))[0]


def test_threads_bit_equal(oracle):  # test_search.cpp:73-98
    rng = np.random.default_rng(61)
    m = rand_model(oracle, rng, 12)
    f = oracle.compute_gradients(rng.integers(0, 256, (40, 40)).astype(float))
    g = ea.PoseGrid(0, 39, 1, 0, 39, 1, 0.0, D(20), D(10))
    base = [(s.score, s.grid_index) for s in oracle.search_topk(m.points, f, g, ea.ScoreParams(3),
                                                                 5, threads=1)]
    for t in (2, 3, 4, 0):
        got = oracle.search_topk(m.points, f, g, ea.ScoreParams(3), 5, threads=t)
        assert [(s.score, s.grid_index) for s in got] == base


def test_score_map_consistency_and_budget(oracle):  # test_search.cpp:100-137
    rng = np.random.default_rng(67)
    m = rand_model(oracle, rng, 10)
    f = oracle.compute_gradients(rng.integers(0, 256, (30, 30)).astype(float))
    g = ea.PoseGrid(5, 24, 1, 5, 24, 1, 0.0, D(10), D(5))
    sm = oracle.score_map(m.points, f, g, ea.ScoreParams(3), 1 << 20)
    d = oracle.exhaustive_search(m.points, f, g, ea.ScoreParams(3))
    assert int(np.argmax(sm)) == d.grid_index and sm.max() == d.score
    with pytest.raises(ea.BudgetError) as e:
        oracle.score_map(m.points, f, ea.PoseGrid(0, 29, 1, 0, 29, 1, 0, 0, 1), ea.ScoreParams(1),
                         100)
    assert "900" in str(e.value) and "100" in str(e.value)


def test_lattice_recovery_and_levels(oracle):  # test_search.cpp:139-234, 264-277
    img, tmpl, _, _ = oracle.compose_scene(ea.SceneSpec(128, 128, "rectangle", 40, (64, 56, 0.0)))
    m = oracle.prepare_model(tmpl)
    f = oracle.compute_gradients(img)
    d = oracle.exhaustive_search(m.points, f, ea.PoseGrid(24, 104, 2, 24, 104, 2, 0, 0, 1),
                                 ea.ScoreParams(3))
    assert d.pose.astuple()[:2] == (64.0, 56.0) and d.score >= 0.95
    flat = np.full((96, 96), 180.0)
    t32 = oracle.render_template("rectangle", 32)
    cfg = ea.SearchConfig(grid=ea.PoseGrid(16, 80, 4, 16, 80, 4, 0, 0, 1), num_levels=2)
    out = oracle.coarse_to_fine(oracle.build_pyramid(t32, 2), oracle.build_pyramid(flat, 2), cfg)
    assert not out.found and out.score < 0.5
    pyr = oracle.build_pyramid(np.full((64, 64), 127.0), 2)
    with pytest.raises(ea.EmptyModelError, match="level 0"):
        oracle.prepare_levels(pyr, pyr, cfg)


def test_topk_monotone(oracle):  # test_search.cpp:236-262
    img, tmpl, _, _ = oracle.compose_scene(ea.SceneSpec(160, 160, "l_bracket", 48,
                                                        (80, 76, D(22)), 14, 99))
    cfg = ea.SearchConfig(grid=ea.PoseGrid(40, 120, 6, 40, 120, 6, 0.0, D(45), D(5)),
                          num_levels=2)
    tp, wp = oracle.build_pyramid(tmpl, 2), oracle.build_pyramid(img, 2)
    prev = -2.0
    for k in (1, 3, 6):
        cfg.topk = k
        s = oracle.coarse_to_fine(tp, wp, cfg).score
        assert s >= prev
        prev = s


# ---- merge (search.cpp:130-139), product host code ---------------------------------------------
def test_merge_topk_host():
    rng = np.random.default_rng(5)
    items = [ea.ScoredPose(float(rng.choice([0.5, 0.25, 0.75])), int(i), ea.Pose(i, 0, 0))
             for i in rng.permutation(40)]
    got = ea.merge_topk(items, 7)
    want = sorted(items, key=lambda s: (-s.score, s.grid_index))[:7]
    assert [(s.score, s.grid_index) for s in got] == [(s.score, s.grid_index) for s in want]
    with pytest.raises(ea.InvalidArgument):
        ea.merge_topk(items, 0)
