"""Golden-fixture checks shared by the oracle (CPU) and the CUDA path (GPU).

The fixtures come from the reference itself (tests/golden/make_golden.py).
Each implementation is wrapped in an adapter exposing one surface.
"""
import hashlib
import json
import os

import numpy as np

from paper_2112_05576_b200 import abi

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    with open(os.path.join(HERE, "golden.json")) as f:
        meta = json.load(f)
    arrays = dict(np.load(os.path.join(HERE, "golden.npz")))
    return meta, arrays


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def scored(lst):
    return [[s.score, int(s.grid_index), s.pose.ux, s.pose.uy, s.pose.theta] for s in lst]


def outcome(o):
    return {"found": bool(o.found), "pose": list(o.pose.astuple()), "score": o.score,
            "grid_index": int(o.grid_index),
            "trace": [[lvl, list(p), sc] for (lvl, p, sc) in o.level_trace()]}


def spec_of(d):
    d = dict(d)
    for k in ("true_pose", "illumination", "occluder"):
        if k in d and d[k] is not None:
            d[k] = tuple(d[k])
    return abi.SceneSpec(**d)


class OracleAdapter:
    def __init__(self, o):
        self.o = o

    def compose_scene(self, spec):
        return self.o.compose_scene(spec)

    def gradients(self, img):
        return self.o.compute_gradients(img)

    def pyramid(self, img, L):
        return self.o.build_pyramid(img, L)

    def model(self, tmpl):
        f = self.o.compute_gradients(tmpl)
        th = self.o.default_thresholds(f)
        return th, self.o.extract_edge_model(f, th, 0)

    def topk(self, pts, field, grid, params, k):
        return self.o.search_topk(pts, field, grid, params, k)

    def score_map(self, pts, field, grid, params):
        return self.o.score_map(pts, field, grid, params, 1 << 20)

    def c2f(self, tmpl, img, cfg):
        L = cfg.num_levels
        return self.o.coarse_to_fine(self.o.build_pyramid(tmpl, L), self.o.build_pyramid(img, L),
                                     cfg)


class ProductAdapter:
    """The CUDA path (device gradients/pyramids/search) + host template side."""

    def __init__(self, ea):
        self.ea = ea

    def compose_scene(self, spec):
        return self.ea.compose_scene(spec)

    def gradients(self, img):
        return tuple(self.ea.compute_gradients(img))

    def pyramid(self, img, L):
        return self.ea.build_pyramid(img, L)

    def model(self, tmpl):
        f = self.ea.compute_gradients(tmpl)
        th = self.ea.default_thresholds(f)
        return th, self.ea.extract_edge_model(f, th, 0)

    def topk(self, pts, field, grid, params, k):
        return self.ea.search_topk(self.ea.EdgeModel(pts), field, grid, params, k=k)

    def score_map(self, pts, field, grid, params):
        return self.ea.score_map(self.ea.EdgeModel(pts), field, grid, params, 1 << 20)

    def c2f(self, tmpl, img, cfg):
        return self.ea.Detector(tmpl, cfg).detect(img)


def check_scenes(impl):
    meta, arr = load()
    for name, m in meta["scenes"].items():
        canvas, tmpl, pose, occ = impl.compose_scene(spec_of(m["spec"]))
        assert np.array_equal(canvas, arr[f"scene_{name}"]), name
        assert np.array_equal(tmpl, arr[f"template_{name}"]), name
        assert list(pose) == m["truth_pose"] and occ == m["occluded_fraction"], name


def check_fields(impl):
    meta, arr = load()
    for name, m in meta["scenes"].items():
        canvas = arr[f"scene_{name}"]
        gx, gy, mag = impl.gradients(canvas)
        assert (sha(gx), sha(gy), sha(mag)) == (m["sha_gx"], m["sha_gy"], m["sha_mag"]), name
        pyr = impl.pyramid(canvas, m["pyramid_levels"])
        assert [sha(l) for l in pyr] == m["sha_pyramid"], name
        th, model = impl.model(arr[f"template_{name}"])
        assert list(th) == m["thresholds"], name
        assert np.array_equal(model.points, arr[f"model_{name}"]), name
        assert [model.centroid_x, model.centroid_y] == m["centroid"], name
    for width in (3, 4, 5, 8, 9, 17, 64, 113):
        got = np.stack(impl.gradients(arr[f"sobel_in_{width}"]))
        assert np.array_equal(got, arr[f"sobel_out_{width}"]), width


def check_searches(impl):
    meta, arr = load()
    for name, m in meta["searches"].items():
        sc = m["scene"]
        pts = arr[f"model_{sc}"]
        field = impl.gradients(arr[f"scene_{sc}"])
        params = abi.ScoreParams(m["nb"], m["polarity"])
        got = impl.topk(pts, field, abi.PoseGrid(*m["grid"]), params, m["k"])
        assert scored(got) == m["topk"], name
        sm = impl.score_map(pts, field, abi.PoseGrid(*m["scoremap_grid"]), params)
        assert np.array_equal(sm, arr[f"scoremap_{name}"]), name


def check_c2f(impl):
    meta, arr = load()
    for name, m in meta["c2f"].items():
        sc = m["scene"]
        cfg = abi.SearchConfig(grid=abi.PoseGrid(*m["grid"]), num_levels=m["num_levels"],
                               score_params=abi.ScoreParams(3), topk=m["topk"],
                               min_score=m["min_score"])
        o = impl.c2f(arr[f"template_{sc}"], arr[f"scene_{sc}"], cfg)
        assert outcome(o) == m["outcome"], name
