"""Model windows above 32. The reference accepts any even W (validate_config,
pipeline.cpp:27-42); the fp32 product kernel holds a window row per warp (W <= 32), so
larger windows run on the generic fp64 kernel for both compute modes (state in shared
memory, or in a global-memory slab once it no longer fits: W >= 68 for RL-JSDE, W >= 74
for L-JSDE). Parity against the unmodified reference (oracle/_ref), same bars as
test_gpu_parity.py / test_gpu_ljsde.py: max-abs <= 1e-9 vs the reference, and the
reference's own L <-> RL equivalence bar (1e-6) where the reference is too slow to run.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inputs(tq, rows, period, seed):
    gt = tq.synthetic_image(rows, rows, seed)
    pat = tq.generate_pattern(7, period)
    return gt, pat, tq.simulate_measurement(gt, pat)


@pytest.mark.parametrize("W,rows", [(36, 72), (40, 80)])
def test_large_window_matches_reference(tq, ref, need_gpu, W, rows):
    _, pat, frame = _inputs(tq, rows, 4, 70 + W)
    want, wrep = ref.reconstruct(frame, pat.opaque, 4, window=W, iterations=30, clip=False,
                                 threads=0)
    for compute in (tq.COMPUTE_FP64, tq.COMPUTE_FP32):  # fp32 requests are served in fp64 here
        cfg = tq.ReconstructionConfig(window=W, max_iterations=30, clip_output=False,
                                      compute=compute)
        rep = tq.reconstruct(frame, pat, cfg)
        assert np.abs(rep.output - want).max() <= 1e-9
        assert rep.blocks_processed == wrep.blocks
        assert rep.classes_total == wrep.classes_total


def test_large_window_ljsde_matches_reference(tq, ref, need_gpu):
    _, pat, frame = _inputs(tq, 72, 4, 106)
    want, _ = ref.reconstruct_algo(frame, pat.opaque, 4, "ljsde", window=36, iterations=6)
    cfg = tq.ReconstructionConfig(window=36, max_iterations=6, clip_output=False,
                                  algorithm=tq.ALGO_LJSDE)
    rep = tq.reconstruct(frame, pat, cfg)
    assert np.abs(rep.output - want).max() <= 1e-9


@pytest.mark.parametrize("algo", ["rljsde", "ljsde"])
def test_global_state_path_matches_reference(tq, ref, need_gpu, monkeypatch, algo):
    """The global-memory state path (taken for W >= 68 / 74) forced at W = 16."""
    monkeypatch.setenv("TQSB_FORCE_GLOBAL_STATE", "1")
    _, pat, frame = _inputs(tq, 48, 8, 48)
    if algo == "rljsde":
        want, _ = ref.reconstruct(frame, pat.opaque, 8, window=16, iterations=40, clip=False)
        cfg = tq.ReconstructionConfig(window=16, max_iterations=40, clip_output=False,
                                      compute=tq.COMPUTE_FP64)
    else:
        want, _ = ref.reconstruct_algo(frame, pat.opaque, 8, "ljsde", window=16, iterations=12)
        cfg = tq.ReconstructionConfig(window=16, max_iterations=12, clip_output=False,
                                      algorithm=tq.ALGO_LJSDE)
    rep = tq.reconstruct(frame, pat, cfg)
    assert np.abs(rep.output - want).max() <= 1e-9


def test_window_76_global_state_l_vs_rl(tq, need_gpu):
    """W = 76 (both kernels keep their state in global memory): the device L-JSDE and
    RL-JSDE agree to the reference's L <-> RL bar (bench, pipeline.cpp:258-329)."""
    gt, pat, frame = _inputs(tq, 80, 4, 176)
    common = dict(window=76, max_iterations=8, clip_output=False)
    rl = tq.reconstruct(frame, pat, tq.ReconstructionConfig(compute=tq.COMPUTE_FP64, **common))
    lj = tq.reconstruct(frame, pat, tq.ReconstructionConfig(algorithm=tq.ALGO_LJSDE, **common))
    assert np.isfinite(rl.output).all()
    assert np.abs(rl.output - lj.output).max() <= 1e-6
    assert 10 * np.log10(1.0 / np.mean((rl.output - gt) ** 2)) > 15
