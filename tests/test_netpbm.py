"""Netpbm codecs and the detection overlay (host code, CPU): byte-identical
to the reference's load_pgm / save_pgm / save_ppm / luminance_to_byte
(image.cpp:26-219, run from oracle/_ref) including every parse error's
message and byte offset; the overlay equals the scorer's own projection."""
import math

import numpy as np
import pytest

import paper_2112_05576_b200 as ea
from paper_2112_05576_b200 import abi


def same_error(fa, fb):
    ea_exc = ref_exc = None
    try:
        a = fa()
    except ea.Error as e:
        ea_exc = e
    try:
        b = fb()
    except ea.Error as e:
        ref_exc = e
    assert (ea_exc is None) == (ref_exc is None), (ea_exc, ref_exc)
    if ea_exc is not None:
        assert type(ea_exc) is type(ref_exc)
        assert str(ea_exc) == str(ref_exc)
        assert getattr(ea_exc, "value", None) == getattr(ref_exc, "value", None)
        return None
    return a, b


PGMS = [
    b"P2\n3 2\n255\n0 1 2\n253 254 255\n",
    b"P2 # comment\n# another\n 4 1 9 0 9 3 4",
    b"P5\n2 2\n255\n\x00\x7f\x80\xff",
    b"P5 2 1 200\n\x05\xc8",
    b"P5\n1 1\n255\n\x00extra",
    b"",
    b"X5\n1 1\n255\n\x00",
    b"P6\n1 1\n255\n\x00\x00\x00",
    b"P2\n",
    b"P2\n3",
    b"P2 a 2 255",
    b"P2 2000000 1 255",
    b"P2 0 1 255",
    b"P2 1 1 0",
    b"P2 1 1 256 7",
    b"P5 1 1 255",
    b"P5 1 1 255x\x00",
    b"P5 2 2 255\n\x00\x00\x00",
    b"P5 2 1 100\n\x05\xc8",
    b"P2 2 1 100 5 101",
    b"P2 2 1 255 5",
    b"P2 1 1 255 99999999999",
]


@pytest.mark.parametrize("i", range(len(PGMS)))
def test_load_pgm_matches_reference(ref, i):
    r = same_error(lambda: ea.load_pgm(PGMS[i]), lambda: ref.load_pgm(PGMS[i]))
    if r is not None:
        assert np.array_equal(r[0], r[1])


def test_save_pgm_ppm_match_reference(ref):
    rng = np.random.default_rng(3)
    img = rng.uniform(-20, 280, size=(17, 23))
    img[0, :6] = [0.5, 1.5, 254.5, 255.0, float("nan"), -0.0]
    assert ea.save_pgm(img) == ref.save_pgm(img)
    overlay = [(0, 0), (22, 16), (5, 7), (-1, 3), (23, 0), (4, 17), (5, 7)]
    for color in [(255, 0, 0), (1, 2, 3)]:
        assert ea.save_ppm(img, overlay, color) == ref.save_ppm(img, overlay, color)
    assert ea.save_ppm(img, [], (9, 9, 9)) == ref.save_ppm(img, [], (9, 9, 9))
    for v in (-1.0, 0.0, 0.49999999999999994, 0.5, 127.5, 254.49, 254.5, 1e300, float("nan")):
        assert ea.luminance_to_byte(v) == ref.luminance_to_byte(v)


def test_pgm_round_trip():
    img = np.arange(24.0).reshape(4, 6) * 10
    assert np.array_equal(ea.load_pgm(ea.save_pgm(img)), np.clip(np.floor(img + 0.5), 0, 255))


def test_overlay_points_is_the_scorer_projection(oracle):
    m = oracle.prepare_model(oracle.render_template("l_bracket", 40))
    for pose in [(50.0, 40.0, 0.3), (10.25, 99.5, abi.deg_to_rad(270)), (0.0, 0.0, 0.0)]:
        got = ea.overlay_points(m, pose)
        px, py, _, _ = oracle.rotate_model(m.points, pose[2])
        want = np.stack([np.floor((px + pose[0]) + 0.5), np.floor((py + pose[1]) + 0.5)], 1)
        assert np.array_equal(got, want.astype(np.int32))


def test_detect_result_json_keys():
    import json
    o = abi.Outcome()
    o.found, o.n_trace, o.score = 1, 2, 0.875
    o.pose = abi.Pose(10.5, 20.25, math.pi / 2)
    o.trace[0].level, o.trace[0].pose, o.trace[0].score = 1, abi.Pose(5.0, 10.0, math.pi / 2), 0.9
    o.trace[1].level, o.trace[1].pose, o.trace[1].score = 0, o.pose, 0.875
    d = json.loads(ea.detect_result_json(o, 120, 0.87))
    assert list(d) == ["pose", "score", "n_model_points", "elapsed_ms", "backend", "level_trace"]
    assert d["pose"] == {"x": 10.5, "y": 20.25, "theta_deg": 90.0}
    assert [t["level"] for t in d["level_trace"]] == [1, 0]
    assert d["level_trace"][0]["theta_deg"] == 90.0


def test_bench_csv_format():
    """BenchRow CSV (SPEC.md cmd_bench): the exact header, one row per
    sample x backend x rep, elapsed_ms > 0 enforced, quoting of names."""
    import paper_2112_05576_b200 as ea
    rows = [{"sample": s, "backend": b, "workers": 0, "run": r, "elapsed_ms": 1.25 + r}
            for s in ("a", "b,c") for b in ("cuda",) for r in range(2)]
    text = ea.bench_csv(rows)
    lines = text.splitlines()
    assert lines[0] == "sample,backend,workers,run,elapsed_ms"
    assert len(lines) == 1 + 4
    assert lines[1] == "a,cuda,0,0,1.250000"
    assert lines[3] == '"b,c",cuda,0,0,1.250000'
    import pytest
    with pytest.raises(ValueError):
        ea.bench_csv([{"sample": "x", "backend": "cuda", "workers": 0, "run": 0,
                       "elapsed_ms": 0.0}])
