"""The CPU oracle (oracle/tqs_oracle.c) pinned against the unmodified reference
(oracle/_ref) and the committed golden fixtures (tests/golden/golden.npz).
Mirrors the reference's own pins (test_grid/test_basis/test_rljsde/test_pipeline)."""
import numpy as np
import pytest


def test_pattern_matches_reference_and_golden(orc, golden):
    for key, want in golden.items():
        if not key.startswith("pattern_s"):
            continue
        seed, P = key[len("pattern_s"):].split("_p")
        got = orc.generate_pattern(int(seed), int(P), 2 if int(P) % 4 else 4)
        np.testing.assert_array_equal(got, want)


def test_pattern_validation(orc):
    with pytest.raises(ValueError):
        orc.generate_pattern(1, 6, 4)  # period not divisible by block (grid.cpp:11-12)
    with pytest.raises(ValueError):
        orc.generate_pattern(1, 2, 2)  # period < 4 (grid.cpp:9-10)


def test_synthetic_and_simulate_bitwise(orc, golden):
    img = orc.synthetic_image(64, 64, 8)
    np.testing.assert_array_equal(img, golden["synthetic_64_s8"])
    assert img.min() >= 0.02 - 1e-15 and img.max() <= 0.98 + 1e-15
    frame = orc.simulate(img, golden["pattern_s7_p32"], 32)
    np.testing.assert_array_equal(frame, golden["frame_64_s8_p32"])


def test_frequency_weights_symmetric(orc, ref):
    q = orc.frequency_weights(32)
    np.testing.assert_array_equal(q, ref.frequency_weights(32))
    Q = q.reshape(32, 32)
    # bitwise symmetric q(k) = q(-k) (test_basis.cpp:239-243)
    neg = Q[(-np.arange(32)) % 32][:, (-np.arange(32)) % 32]
    np.testing.assert_array_equal(Q, neg)
    assert q[0] == max(q) and (q > 0).all()


def test_tables_match_golden(orc, golden):
    t = orc.tables(golden["pattern_s5_p8"], 8, 3, 5, 8)
    np.testing.assert_array_equal(t["b"], golden["tables_w8_p8_s5_o3_5_b"])
    np.testing.assert_array_equal(t["c"], golden["tables_w8_p8_s5_o3_5_c"])
    np.testing.assert_array_equal(t["d"], golden["tables_w8_p8_s5_o3_5_d"])


@pytest.mark.parametrize("W,P,o", [(8, 8, (0, 0)), (8, 8, (3, 5)), (16, 32, (6, 10)),
                                   (32, 8, (2, 6))])
def test_tables_match_reference(orc, ref, W, P, o):
    pat = ref.generate_pattern(7, P, 2)
    a = orc.tables(pat, P, o[0], o[1], W)
    b = ref.precompute(pat, P, o[0], o[1], W)
    assert a["L"] == b["L"]
    np.testing.assert_array_equal(a["b"], b["b"])
    np.testing.assert_array_equal(a["c"], b["c"])
    np.testing.assert_array_equal(a["d"], b["d"])


def test_table_structure(orc):
    """Hermitian C mirrored bitwise, D = Re diag C, D >= 0 (test_rljsde.cpp:129-145)."""
    pat = orc.generate_pattern(103, 8, 2)
    t = orc.tables(pat, 8, 1, 2, 8)
    C = t["c"].reshape(64, 64)  # [uk, sk]
    off = ~np.eye(64, dtype=bool)
    np.testing.assert_array_equal(C.real, C.real.T)
    np.testing.assert_array_equal(C.imag[off], -C.imag.T[off])
    assert np.abs(np.diag(C).imag).max() < 1e-14
    np.testing.assert_array_equal(t["d"], np.diag(C).real)
    assert (t["d"] >= 0).all()


@pytest.mark.parametrize("W,L", [(8, 16), (32, 256)])
def test_dc_energy_equals_local_count_under_unit_weights(orc, W, L):
    """test_rljsde.cpp:147-164: decay 1 gives unit weights, D[DC] == L exactly."""
    pat = orc.generate_pattern(7 if W == 32 else 5, 32 if W == 32 else 8, 4 if W == 32 else 2)
    t = orc.tables(pat, 32 if W == 32 else 8, 0, 0, W, decay=1.0)
    assert t["L"] == L
    assert t["d"][0] == float(L)


def test_block_trace_matches_reference(orc, ref, golden):
    pat8 = golden["pattern_s7_p8"]
    frame = golden["frame_128_s301_p8"]
    y = orc.gather(frame, 14, 14, 32)
    t = orc.tables(pat8, 8, 14, 14, 32)
    q = orc.frequency_weights(32)
    picks, gd, win = orc.block(t, q, y, 32)
    np.testing.assert_array_equal(picks, golden["trace_128_s301_p8_o14_14_picks"])
    np.testing.assert_array_equal(gd, golden["trace_128_s301_p8_o14_14_gd"])
    np.testing.assert_array_equal(win.ravel(), golden["trace_128_s301_p8_o14_14_window"].ravel())


def test_census_matches_reference_pins(orc):
    """test_pipeline.cpp:169-190: 64x64, P = 32."""
    c = orc.census(32, 32, window=32, block=4, period=32)
    assert (c["blocks"], c["classes_total"], c["classes_interior"]) == (256, 81, 64)
    c = orc.census(32, 32, window=16, block=4, period=32)
    assert (c["classes_total"], c["classes_interior"]) == (100, 64)


def test_reconstruct_matches_golden(orc, golden):
    frame = golden["frame_64_s8_p32"]
    out = orc.reconstruct(frame, golden["pattern_s7_p32"], 32, window=16, iterations=100,
                          clip=False)
    np.testing.assert_array_equal(out, golden["recon_64_s8_p32_w16_it100"])


@pytest.mark.slow
def test_reconstruct_default_config_matches_golden(orc, golden):
    """The BASELINE oracle config (128x128, P = 8, W = 32, nu = 200)."""
    out = orc.reconstruct(golden["frame_128_s301_p8"], golden["pattern_s7_p8"], 8, clip=False)
    np.testing.assert_array_equal(out, golden["recon_128_s301_p8_default_noclip"])


def test_constant_image_one_step(orc):
    """test_pipeline.cpp:149-167: constant 0.6, gamma = 1, nu = 1 -> 0.6 everywhere."""
    pat = orc.generate_pattern(7, 32)
    img = np.full((64, 64), 0.6)
    frame = orc.simulate(img, pat, 32)
    out = orc.reconstruct(frame, pat, 32, window=16, iterations=1, step=1.0, clip=False)
    np.testing.assert_allclose(out, 0.6, rtol=1e-10, atol=0)
    assert orc.psnr(img, out) >= 60


def test_psnr_reference_points(orc):
    a, b = np.zeros((4, 4)), np.ones((4, 4))
    assert orc.psnr(a, b) == 0.0
    assert orc.psnr(a, a) == float("inf")
    assert abs(orc.psnr(np.full((4, 4), 0.5), np.full((4, 4), 0.51)) - 40.0) < 1e-9
