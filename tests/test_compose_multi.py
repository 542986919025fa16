"""Multi-stamp scene composer (ea_compose_multi, the cfg5 input generator;
host code, runs on CPU).  One stamp reproduces compose_scene, which
tests/test_golden.py pins to the reference's own scenes."""
import numpy as np
import pytest

import paper_2112_05576_b200 as ea
from paper_2112_05576_b200 import abi

D = abi.deg_to_rad


@pytest.mark.parametrize("tid,size,pose,occ,illum,sigma", [
    ("l_bracket", 40, (48.0, 40.0, D(33)), None, (1.0, 0.0, 1.0), 0.0),
    ("rectangle", 64, (90.5, 70.25, D(200)), (20, 30, 40, 25, 10.0), (1.7, -30.0, 1.2), 2.0),
    ("ring", 32, (50.0, 50.0, 0.0), None, (0.8, 5.0, 1.0), 1.0),
    ("cross", 48, (70.0, 60.0, D(359.5)), (60, 50, 30, 30, 250.0), (1.0, 0.0, 0.7), 0.0),
])
def test_one_stamp_equals_compose_scene(tid, size, pose, occ, illum, sigma):
    spec = abi.SceneSpec(160, 120, tid, size, pose, 30, 77, occ, illum, sigma, 5)
    canvas, _, _, _ = ea.compose_scene(spec)
    multi = ea.compose_multi(spec, [(tid, size, pose)])
    assert np.array_equal(canvas, multi)


def test_disjoint_stamps_commute_and_land():
    spec = abi.SceneSpec(300, 200, "rectangle", 0, (0, 0, 0), 20, 9, None, (1.0, 0.0, 1.0), 0.0, 0)
    a = ("l_bracket", 48, (70.0, 100.0, D(10)))
    b = ("cross", 64, (220.0, 100.0, D(80)))
    ab = ea.compose_multi(spec, [a, b])
    ba = ea.compose_multi(spec, [b, a])
    assert np.array_equal(ab, ba)
    # each stamp alone changes only its own half of the canvas
    only_a = ea.compose_multi(spec, [a])
    only_b = ea.compose_multi(spec, [b])
    bg = ea.compose_multi(spec, [])
    assert np.array_equal(ab[:, :150], only_a[:, :150])
    assert np.array_equal(ab[:, 150:], only_b[:, 150:])
    assert not np.array_equal(only_a, bg) and not np.array_equal(only_b, bg)


def test_overlapping_stamps_union_ink():
    """Only ink pixels land (synth.cpp:238-241) and every template uses the
    same ink, so overlapping stamps paint the union of their shapes."""
    spec = abi.SceneSpec(120, 120, "rectangle", 0, (0, 0, 0), 0, 0, None, (1.0, 0.0, 1.0), 0.0, 0)
    a = ("rectangle", 64, (60.0, 60.0, 0.0))
    b = ("cross", 64, (60.0, 60.0, 0.0))
    ab = ea.compose_multi(spec, [a, b])
    assert np.array_equal(ab, ea.compose_multi(spec, [b, a]))
    ink_a = ea.compose_multi(spec, [a]) != 200.0
    ink_b = ea.compose_multi(spec, [b]) != 200.0
    assert np.array_equal(ab != 200.0, ink_a | ink_b)


def test_stamp_off_canvas_raises():
    spec = abi.SceneSpec(100, 100, "rectangle", 0, (0, 0, 0), 0, 0, None, (1.0, 0.0, 1.0), 0.0, 0)
    with pytest.raises(ea.GeometryError, match="leaves the canvas"):
        ea.compose_multi(spec, [("ring", 32, (50, 50, 0.0)), ("ring", 64, (95.0, 50.0, 0.0))])
    with pytest.raises(ea.SizeError):
        ea.compose_multi(spec, [("ring", 8, (50, 50, 0.0))])
