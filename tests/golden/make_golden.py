"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

    make -C oracle ref && python tests/golden/make_golden.py

Runs oracle/_ref/libedgealign_ref.so (the reference compiled from its own
sources under /root/reference/proj/src, behind oracle/ref_shim.cpp) on seeded
inputs and writes:

  golden.npz   small arrays (scenes, templates, edge models, score maps, ...)
  golden.json  scalar results (top-k lists, outcomes, sha256 of large arrays)

The fixtures pin the C oracle (tests/test_golden.py, CPU) and the CUDA path
(tests/test_gpu_golden.py, GPU) without needing /root/reference at run time.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import ReferenceLib  # noqa: E402
from paper_2112_05576_b200 import abi  # noqa: E402

D = abi.deg_to_rad


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def scored(lst):
    return [[s.score, int(s.grid_index), s.pose.ux, s.pose.uy, s.pose.theta] for s in lst]


def outcome(o):
    return {"found": bool(o.found), "pose": list(o.pose.astuple()), "score": o.score,
            "grid_index": int(o.grid_index),
            "trace": [[lvl, list(p), sc] for (lvl, p, sc) in o.level_trace()]}


# Scenes: the reference's own test geometries (test_search.cpp:139-262) plus a
# degraded one (occluder + illumination + noise, like BASELINE configs[1]).
SCENES = {
    "lattice_rect": dict(canvas_width=128, canvas_height=128, template_id="rectangle",
                         template_size=40, true_pose=(64, 56, 0.0)),
    "cross_1level": dict(canvas_width=96, canvas_height=96, template_id="cross",
                         template_size=32, true_pose=(48, 48, 0.0)),
    "bracket_clutter": dict(canvas_width=160, canvas_height=160, template_id="l_bracket",
                            template_size=48, true_pose=(80, 76, D(22)), clutter_segments=14,
                            clutter_seed=99),
    "ring_degraded": dict(canvas_width=144, canvas_height=112, template_id="ring",
                          template_size=40, true_pose=(70, 60, D(10)), clutter_segments=20,
                          clutter_seed=5, occluder=(60, 40, 20, 30, 200.0),
                          illumination=(1.7, -30.0, 1.2), noise_sigma=2.0, noise_seed=13),
}

SEARCHES = {
    # name: (scene, grid, nb, polarity, k)
    "lattice_rect": ("lattice_rect", (24, 104, 2, 24, 104, 2, 0.0, 0.0, 1.0), 3, 0, 5),
    "bracket_full": ("bracket_clutter", (0, 159, 1, 0, 159, 1, 0.0, D(357), D(3)), 3, 0, 7),
    "bracket_ignore": ("bracket_clutter", (20, 140, 1, 20, 140, 1, 0.0, D(40), D(4)), 3, 1, 5),
    "ring_nb5": ("ring_degraded", (10, 130, 1, 10, 100, 1, -0.2, 0.3, D(5)), 5, 0, 5),
    "ring_general": ("ring_degraded", (10.5, 130, 1.5, 9.25, 100, 1.25, 0.0, 0.3, 0.1), 3, 0, 5),
}

C2F = {
    # name: (scene, grid, num_levels, topk, min_score)
    "cross_1level": ("cross_1level", (24, 72, 2, 24, 72, 2, 0.0, 0.0, 1.0), 1, 5, 0.5),
    "bracket_2level": ("bracket_clutter", (40, 120, 6, 40, 120, 6, 0.0, D(45), D(5)), 2, 6, 0.5),
    "bracket_3level": ("bracket_clutter", (0, 159, 4, 0, 159, 4, 0.0, D(358), D(2)), 3, 5, 0.5),
    "ring_2level": ("ring_degraded", (0, 143, 2, 0, 111, 2, 0.0, D(90), D(3)), 2, 5, 0.4),
}


def main():
    ref = ReferenceLib()
    arrays, meta = {}, {"scenes": {}, "searches": {}, "c2f": {}, "kernels": {}}
    models = {}
    for name, kw in SCENES.items():
        spec = abi.SceneSpec(**kw)
        canvas, tmpl, pose, occ = ref.compose_scene(spec)
        arrays[f"scene_{name}"] = canvas
        arrays[f"template_{name}"] = tmpl
        field = ref.compute_gradients(canvas)
        tfield = ref.compute_gradients(tmpl)
        th = ref.default_thresholds(tfield)
        model = ref.extract_edge_model(tfield, th, 0)
        models[name] = (model, field)
        arrays[f"model_{name}"] = model.points
        pyr = ref.build_pyramid(canvas, ref.max_pyramid_levels(canvas.shape[1], canvas.shape[0]))
        meta["scenes"][name] = {
            "spec": {k: (list(v) if isinstance(v, tuple) else v) for k, v in kw.items()},
            "truth_pose": list(pose), "occluded_fraction": occ,
            "thresholds": list(th), "centroid": [model.centroid_x, model.centroid_y],
            "sha_gx": sha(field[0]), "sha_gy": sha(field[1]), "sha_mag": sha(field[2]),
            "sha_pyramid": [sha(l) for l in pyr], "pyramid_levels": len(pyr)}
    for name, (sc, g, nb, pol, k) in SEARCHES.items():
        model, field = models[sc]
        grid = abi.PoseGrid(*g)
        params = abi.ScoreParams(nb, pol)
        top = ref.search_topk(model.points, field, grid, params, k)
        meta["searches"][name] = {"scene": sc, "grid": list(g), "nb": nb, "polarity": pol,
                                  "k": k, "topk": scored(top)}
        # a small exact score map around the best pose
        b = top[0].pose
        sg = (b.ux - 2 * g[2], b.ux + 2 * g[2], g[2], b.uy - 2 * g[5], b.uy + 2 * g[5], g[5],
              b.theta - g[8], b.theta + g[8], g[8])
        arrays[f"scoremap_{name}"] = ref.score_map(model.points, field, abi.PoseGrid(*sg), params,
                                                   1 << 20)
        meta["searches"][name]["scoremap_grid"] = list(sg)
    for name, (sc, g, L, k, ms) in C2F.items():
        canvas, tmpl = arrays[f"scene_{sc}"], arrays[f"template_{sc}"]
        cfg = abi.SearchConfig(grid=abi.PoseGrid(*g), num_levels=L, score_params=abi.ScoreParams(3),
                               topk=k, min_score=ms)
        o = ref.coarse_to_fine(ref.build_pyramid(tmpl, L), ref.build_pyramid(canvas, L), cfg)
        meta["c2f"][name] = {"scene": sc, "grid": list(g), "num_levels": L, "topk": k,
                             "min_score": ms, "outcome": outcome(o)}
    # Kernel KATs (test_kernels.cpp:30-107 shapes), scalar ISA of the reference
    rng = np.random.default_rng(42)
    for width in (3, 4, 5, 8, 9, 17, 64, 113):
        rows = rng.uniform(-500, 500, size=(3, width))
        img = np.vstack([rows, rows[:1]])  # 4 rows; row 1 is the Sobel middle row
        g = ref.compute_gradients(img) if width >= 3 else None
        arrays[f"sobel_in_{width}"] = img
        arrays[f"sobel_out_{width}"] = np.stack(g)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"), len(arrays), "arrays")


if __name__ == "__main__":
    main()
