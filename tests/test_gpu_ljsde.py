"""L-JSDE baseline on the device (ljsde.cpp:131-185) against the
unmodified reference: per-block greedy paths, whole reconstructions, the energy stop,
and the reference's L <-> RL equivalence bar (bench, pipeline.cpp:258-329)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [120, 121, 122, 123])
def test_ljsde_paths_match_reference(tq, ref, need_gpu, seed):
    """random W=8 windows (odd origins give L < W^2/4), 30 iterations: identical picks."""
    rng = np.random.default_rng(seed)
    pat = tq.generate_pattern(int(rng.integers(1 << 30)), 8, 2)
    o = (int(rng.integers(8)), int(rng.integers(8)))
    L = ref.precompute(pat.opaque, 8, o[0], o[1], 8)["L"]
    y = rng.random(L)
    cfg = tq.ReconstructionConfig(window=8, block=2, max_iterations=30, algorithm=tq.ALGO_LJSDE)
    with tq.Plan(pat, cfg) as plan:
        picks, gd, win = plan.block_trace(o[0], o[1], y)
    rp, rgd, rwin = ref.ljsde_trace(pat.opaque, 8, o[0], o[1], 8, y, iterations=30)
    np.testing.assert_array_equal(picks, rp)
    assert np.max(np.abs(gd - rgd)) < 1e-12
    assert np.max(np.abs(win - rwin)) < 1e-12


def test_ljsde_default_window_path(tq, ref, need_gpu):
    """W = 32 interior window of the 128^2 acceptance image, 40 iterations."""
    gt = tq.synthetic_image(128, 128, 301)
    pat = tq.generate_pattern(7, 8)
    frame = tq.simulate_measurement(gt, pat)
    o = (14, 14)
    L = ref.precompute(pat.opaque, 8, o[0], o[1], 32)["L"]
    r0, c0 = (o[0] + 1) // 2, (o[1] + 1) // 2
    n = int(np.sqrt(L))
    y = frame[r0:r0 + n, c0:c0 + n].ravel()
    cfg = tq.ReconstructionConfig(max_iterations=40, algorithm=tq.ALGO_LJSDE)
    with tq.Plan(pat, cfg) as plan:
        picks, gd, win = plan.block_trace(o[0], o[1], y)
    rp, rgd, rwin = ref.ljsde_trace(pat.opaque, 8, o[0], o[1], 32, y, iterations=40)
    np.testing.assert_array_equal(picks, rp)
    assert np.max(np.abs(win - rwin)) < 1e-11


def test_ljsde_energy_stop_matches_reference(tq, ref, need_gpu):
    """earlyStop (basis.hpp:80-81): the block ends once sum w |r|^2 < scale * L."""
    rng = np.random.default_rng(5)
    pat = tq.generate_pattern(11, 8, 2)
    L = ref.precompute(pat.opaque, 8, 2, 2, 8)["L"]
    y = rng.random(L)
    for scale in (1e-2, 1e-4, 1e30):
        cfg = tq.ReconstructionConfig(window=8, block=2, max_iterations=60,
                                      algorithm=tq.ALGO_LJSDE, early_stop=True,
                                      early_stop_scale=scale)
        with tq.Plan(pat, cfg) as plan:
            picks, gd, win = plan.block_trace(2, 2, y)
        rp, rgd, rwin = ref.ljsde_trace(pat.opaque, 8, 2, 2, 8, y, iterations=60,
                                        early_stop_scale=scale)
        np.testing.assert_array_equal(picks, rp)
        assert np.max(np.abs(win - rwin)) < 1e-12
        if scale == 1e30:
            assert len(picks) == 1


@pytest.mark.parametrize("rows,W,it,period", [(32, 16, 8, 32), (48, 16, 6, 32), (64, 32, 20, 8)])
def test_ljsde_reconstruct_matches_reference(tq, ref, need_gpu, rows, W, it, period):
    gt = tq.synthetic_image(rows, rows, 60 + rows)
    pat = tq.generate_pattern(7, period)
    frame = tq.simulate_measurement(gt, pat)
    want, _ = ref.reconstruct_algo(frame, pat.opaque, period, "ljsde", window=W, iterations=it)
    cfg = tq.ReconstructionConfig(window=W, max_iterations=it, clip_output=False,
                                  algorithm=tq.ALGO_LJSDE)
    rep = tq.reconstruct(frame, pat, cfg)
    assert np.abs(rep.output - want).max() <= 1e-9
    assert rep.classes_created == 0 and rep.cache_hits == 0 and rep.cache_misses == 0
    # the reference's L <-> RL equivalence bar (bench threshold 1e-6) holds on the device
    rl = tq.reconstruct(frame, pat, tq.ReconstructionConfig(
        window=W, max_iterations=it, clip_output=False, compute=tq.COMPUTE_FP64))
    assert np.abs(rl.output - rep.output).max() <= 1e-6
