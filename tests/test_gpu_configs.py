"""Window / block / period combinations beyond the defaults, through every kernel
instantiation family of the fp32 product path (rank slots NS = 1..16 incl. padded
rank sets such as W = 30, kept-pixel groups PPL = 1/2/8, the 12-warp heavy variants)
and the fp64 parity mode, against the unmodified reference (validate_config's rules,
pipeline.cpp:27-42: B | W, (W - B) even, B | P).

Bars as in test_gpu_parity.py: the fp64 mode is bitwise equal to the reference (it
spells every expression in the reference build's rounding pattern, solve_f64.cu); fp32
product |dPSNR| <= 0.01 dB and max-abs <= 1e-2 vs the reference.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _psnr(ref, est):
    return -10 * np.log10(np.mean((ref - est) ** 2))


@pytest.mark.parametrize("W,B,P,rows", [
    (8, 2, 4, 32),      # NS = 1
    (12, 4, 8, 48),     # NS = 4, padded ranks (K = 144)
    (20, 4, 4, 64),     # NS = 8, padded ranks (K = 400)
    (18, 6, 12, 72),    # B = 6 (PPL = 2), P = 12
    (24, 8, 8, 64),     # NS = 16, PPL = 2, padded ranks (K = 576)
    (30, 2, 4, 64),     # NS = 16, K = 900
    (32, 8, 8, 64),     # default window, B = 8 (12-warp instantiation)
    (16, 16, 16, 48),   # B = W: PPL = 8, no context around the target block
])
def test_config_matches_reference(tq, ref, need_gpu, W, B, P, rows):
    img = tq.synthetic_image(rows, rows + 2 * B, 500 + W + B)
    pat = tq.generate_pattern(11, P, B)
    frame = tq.simulate_measurement(img, pat)
    it = 60
    want, wrep = ref.reconstruct(frame, pat.opaque, P, window=W, block=B, iterations=it,
                                 clip=False, threads=0)
    common = dict(window=W, block=B, max_iterations=it, clip_output=False)
    f64 = tq.reconstruct(frame, pat, tq.ReconstructionConfig(compute=tq.COMPUTE_FP64, **common))
    assert np.array_equal(f64.output, want)
    assert f64.blocks_processed == wrep.blocks
    assert f64.classes_total == wrep.classes_total
    f32 = tq.reconstruct(frame, pat, tq.ReconstructionConfig(compute=tq.COMPUTE_FP32, **common))
    assert np.abs(f32.output - want).max() <= 1e-2
    assert abs(_psnr(img, f32.output) - _psnr(img, want)) <= 0.01
