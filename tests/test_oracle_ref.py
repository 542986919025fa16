"""Pin the C oracle to the reference itself (oracle/_ref, compiled from
/root/reference/proj/src by oracle/Makefile): bit-exact on randomised inputs,
same exceptions and messages.  Skipped when oracle/_ref was not built."""
import numpy as np
import pytest

from paper_2112_05576_b200 import abi
from paper_2112_05576_b200.errors import Error

D = abi.deg_to_rad


def rand_img(rng, w, h, real=True):
    if real:
        return rng.uniform(-40, 300, size=(h, w))
    return rng.integers(0, 256, size=(h, w)).astype(np.float64)


def same_error(f, g):
    """Both raise the same exception class with the same message, or both
    return equal values."""
    try:
        a = f()
    except Error as e:
        with pytest.raises(type(e)) as info:
            g()
        assert str(info.value) == str(e)
        return None
    b = g()
    return a, b


def test_scenes(oracle, ref):
    rng = np.random.default_rng(1)
    for trial in range(25):
        tid = ["rectangle", "ring", "l_bracket", "cross"][trial % 4]
        size = int(rng.integers(16, 80))
        W, H = int(rng.integers(64, 200)), int(rng.integers(64, 200))
        occ = None
        if trial % 3 == 0:
            occ = (int(rng.integers(0, W)), int(rng.integers(0, H)), int(rng.integers(1, 40)),
                   int(rng.integers(1, 40)), float(rng.uniform(0, 255)))
        spec = abi.SceneSpec(W, H, tid, size,
                             (float(rng.uniform(0, W)), float(rng.uniform(0, H)),
                              float(rng.uniform(-4, 4))),
                             int(rng.integers(0, 30)), int(rng.integers(0, 1 << 62)), occ,
                             (float(rng.uniform(0.5, 2)), float(rng.uniform(-40, 40)),
                              float(rng.choice([1.0, 0.7, 1.3]))),
                             float(rng.choice([0.0, 1.5])), int(rng.integers(0, 1000)))
        r = same_error(lambda: oracle.compose_scene(spec), lambda: ref.compose_scene(spec))
        if r:
            (a, b) = r
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            assert a[2:] == b[2:]


def test_fields_pyramids(oracle, ref):
    rng = np.random.default_rng(2)
    for (w, h) in [(3, 3), (4, 9), (17, 5), (64, 47), (200, 150), (2, 2), (1, 7)]:
        img = rand_img(rng, w, h)
        r = same_error(lambda: oracle.compute_gradients(img), lambda: ref.compute_gradients(img))
        if r:
            for x, y in zip(*r):
                assert np.array_equal(x, y)
        r = same_error(lambda: oracle.downsample(img), lambda: ref.downsample(img))
        if r:
            assert np.array_equal(*r)
        L = oracle.max_pyramid_levels(w, h)
        assert L == ref.max_pyramid_levels(w, h)
        for lv in (L, L + 1):
            r = same_error(lambda: oracle.build_pyramid(img, lv), lambda: ref.build_pyramid(img, lv))
            if r:
                assert all(np.array_equal(x, y) for x, y in zip(*r))


def test_edge_models(oracle, ref):
    rng = np.random.default_rng(3)
    for trial in range(30):
        img = rand_img(rng, int(rng.integers(5, 40)), int(rng.integers(5, 40)), trial % 2 == 0)
        f = oracle.compute_gradients(img)
        assert oracle.default_thresholds(f) == ref.default_thresholds(f)
        hi = float(rng.uniform(0, 1500))
        th = (float(rng.uniform(0, hi)), hi) if trial % 5 else (0.0, 0.0)
        r = same_error(lambda: oracle.extract_edge_model(f, th, 2),
                       lambda: ref.extract_edge_model(f, th, 2))
        if r:
            a, b = r
            assert np.array_equal(a.points, b.points)
            assert (a.centroid_x, a.centroid_y) == (b.centroid_x, b.centroid_y)
    flat = oracle.compute_gradients(np.full((9, 9), 55.0))
    same_error(lambda: oracle.extract_edge_model(flat, (0, 0), 0),
               lambda: ref.extract_edge_model(flat, (0, 0), 0))
    same_error(lambda: oracle.extract_edge_model(flat, (2, 1), 0),
               lambda: ref.extract_edge_model(flat, (2, 1), 0))


def test_rotation_and_scores(oracle, ref):
    rng = np.random.default_rng(4)
    m = oracle.prepare_model(oracle.render_template("l_bracket", 40))
    f = oracle.compute_gradients(rand_img(rng, 60, 50))
    for trial in range(200):
        th = float(rng.uniform(-7, 7))
        for x, y in zip(oracle.rotate_model(m.points, th), ref.rotate_model(m.points, th)):
            assert np.array_equal(x, y)
        pose = (float(rng.uniform(-20, 80)), float(rng.uniform(-20, 70)), th)
        p = abi.ScoreParams(int(rng.choice([1, 3, 5, 7])), int(trial % 2))
        assert oracle.pose_score(m.points, pose, f, p) == ref.pose_score(m.points, pose, f, p)
        cx, cy = int(rng.integers(-5, 65)), int(rng.integers(-5, 55))
        dx, dy = np.cos(th), np.sin(th)
        assert oracle.point_vote(dx, dy, f, cx, cy, p) == ref.point_vote(dx, dy, f, cx, cy, p)
    for bad in (abi.ScoreParams(2), abi.ScoreParams(0), abi.ScoreParams(3, 0, 0.0),
                abi.ScoreParams(3, 0, -1.0)):
        same_error(lambda: oracle.pose_score(m.points, (1, 1, 0), f, bad),
                   lambda: ref.pose_score(m.points, (1, 1, 0), f, bad))


@pytest.mark.parametrize("seed", range(6))
def test_search_topk(oracle, ref, seed):
    rng = np.random.default_rng(10 + seed)
    f = oracle.compute_gradients(rand_img(rng, 40, 36, real=False))
    mf = oracle.compute_gradients(rand_img(rng, 12, 12, real=False))
    m = oracle.extract_edge_model(mf, (0.0, 0.0), 0)
    grids = [(0, 39, 1, 0, 35, 1, 0.0, D(30), D(10)), (-3.5, 41, 1.5, 2, 30, 2.5, -1, 1, 0.25),
             (5, 5, 1, 6, 6, 1, 0.2, 0.2, 0.1)]
    g = abi.PoseGrid(*grids[seed % 3])
    p = abi.ScoreParams([1, 3, 5][seed % 3], seed % 2)
    for k in (1, 5, 13):
        a = oracle.search_topk(m.points, f, g, p, k, threads=3)
        b = ref.search_topk(m.points, f, g, p, k)
        assert [(s.score, s.grid_index, s.pose.astuple()) for s in a] == \
               [(s.score, s.grid_index, s.pose.astuple()) for s in b]
    assert np.array_equal(oracle.score_map(m.points, f, g, p, 1 << 20),
                          ref.score_map(m.points, f, g, p, 1 << 20))
    same_error(lambda: oracle.score_map(m.points, f, g, p, 0),
               lambda: ref.score_map(m.points, f, g, p, 0))


@pytest.mark.parametrize("seed", range(4))
def test_coarse_to_fine(oracle, ref, seed):
    rng = np.random.default_rng(20 + seed)
    W, H = 160, 128
    spec = abi.SceneSpec(W, H, ["l_bracket", "rectangle", "cross", "ring"][seed], 48,
                         (80.0, 64.0, float(rng.uniform(0, 6.28))), 10, seed)
    img, tmpl, _, _ = ref.compose_scene(spec)
    L = 1 + seed % 3
    cfg = abi.SearchConfig(grid=abi.PoseGrid(0, W - 1, 1 << (L - 1), 0, H - 1, 1 << (L - 1), 0.0,
                                             D(350), D(10)),
                           num_levels=L, score_params=abi.ScoreParams(3), topk=1 + seed,
                           refine_radius=1 + seed % 2)
    tp, wp = ref.build_pyramid(tmpl, L), ref.build_pyramid(img, L)
    assert oracle.coarse_to_fine(tp, wp, cfg).key() == ref.coarse_to_fine(tp, wp, cfg).key()
    cfg.has_thresholds, cfg.thresholds = 1, abi.EdgeThresholds(30.0, 300.0)
    r = same_error(lambda: oracle.coarse_to_fine(tp, wp, cfg).key(),
                   lambda: ref.coarse_to_fine(tp, wp, cfg).key())
    if r:
        assert r[0] == r[1]
