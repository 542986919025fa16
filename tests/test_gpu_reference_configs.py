"""Parity pinned DIRECTLY to the reference at the BASELINE configs' scale:
the GPU detect against the reference library itself (oracle/_ref: the
reference compiled unmodified from /root/reference/proj/src, its own
coarse_to_fine search.cpp:359-364, Backend::Parallel on every host thread),
not through the C restatement.  Inputs come from the reference's own
compose_scene (synth.cpp:178-300); cfg5's multi-stamp scene has no reference
composer and comes from ea_compose_multi (byte-identical to
compose_scene for one stamp, tests/test_compose_multi.py).  Outcomes are
compared bit for bit: found flag, pose, score, winning grid index and the
per-level trace (Outcome.key()).
"""
import os

import pytest

from paper_2112_05576_b200 import abi

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def ref_cfg(cfg):
    """The same SearchConfig with the reference's Parallel backend."""
    return abi.SearchConfig(grid=cfg.grid, num_levels=cfg.num_levels,
                            score_params=cfg.score_params, topk=cfg.topk,
                            refine_radius=cfg.refine_radius, min_score=cfg.min_score,
                            backend_kind=abi.BACKEND_PARALLEL,
                            worker_count=len(os.sched_getaffinity(0)))


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_detect_equals_reference(ea, ref, name):
    import bench
    img, tmpl, cfg, _ = bench.make_inputs(name, compose=ref.compose_scene)
    L = cfg.num_levels
    want = ref.coarse_to_fine(ref.build_pyramid(tmpl, L), ref.build_pyramid(img, L), ref_cfg(cfg))
    det = ea.Detector(tmpl, cfg)
    assert det.detect(img).key() == want.key()
    assert det.detect_batch([img, img])[1].key() == want.key()


def test_cfg3_sharded_detect_equals_reference(ea, ref):
    """The theta-sharded detect of BASELINE configs[2] (world-1 NCCL
    communicator: input broadcast, slab search, all-gather, merge, root
    refinement, outcome broadcast) == the reference."""
    import bench
    img, tmpl, cfg, _ = bench.make_inputs("cfg3", compose=ref.compose_scene)
    L = cfg.num_levels
    want = ref.coarse_to_fine(ref.build_pyramid(tmpl, L), ref.build_pyramid(img, L), ref_cfg(cfg))
    ctx = ea.Context(0)
    try:
        ctx.comm_init(0, 1, ea.comm_unique_id())
        assert ea.Detector(tmpl, cfg, ctx).detect_sharded(img).key() == want.key()
    finally:
        ctx.close()


def test_cfg5_multi_detect_equals_reference(ea, ref):
    """BASELINE configs[4]: 8 models on one 2592x1944 cluttered scene,
    detect_multi (shared pyramid, region-tiled screening) == the reference's
    coarse_to_fine per model."""
    import bench
    img, tmpls, cfg, _ = bench.make_multi_inputs("cfg5")
    L = cfg.num_levels
    dets = [ea.Detector(t, cfg) for t in tmpls]
    outs = ea.detect_multi(dets, img)
    wp = ref.build_pyramid(img, L)
    rc = ref_cfg(cfg)
    for t, got in zip(tmpls, outs):
        assert got.key() == ref.coarse_to_fine(ref.build_pyramid(t, L), wp, rc).key()
