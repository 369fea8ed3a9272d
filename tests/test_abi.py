"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/tqsb/tqsb.h declares, its host helpers reproduce the reference
bitwise, validation mirrors pipeline.cpp:27-42, and compute entry points fail
loudly (no CPU fallback) when no device is present."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tqsb", "tqsb.h")).read()
    return sorted(set(re.findall(r"\b(tqsb_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(tq):
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(tq.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"libtqsb.so does not export {s}"
    assert set(syms) == set(tq.EXPORTS)


def test_version(tq):
    assert b"sm_100a" in tq.lib.tqsb_version()


def test_host_pattern_image_simulate_match_reference(tq, golden):
    for key, want in golden.items():
        if key.startswith("pattern_s"):
            seed, P = key[len("pattern_s"):].split("_p")
            got = tq.generate_pattern(int(seed), int(P), 2 if int(P) % 4 else 4)
            np.testing.assert_array_equal(got.opaque, want)
    img = tq.synthetic_image(64, 64, 8)
    np.testing.assert_array_equal(img, golden["synthetic_64_s8"])
    pat = tq.QuadrantPattern(32, golden["pattern_s7_p32"])
    np.testing.assert_array_equal(tq.simulate_measurement(img, pat), golden["frame_64_s8_p32"])


def test_host_generators_vs_reference_other_sizes(tq, ref):
    for rows, cols, seed in [(128, 128, 301), (33, 38, 11), (2160 // 8, 3840 // 8, 501)]:
        np.testing.assert_array_equal(tq.synthetic_image(rows, cols, seed),
                                      ref.synthetic_image(rows, cols, seed))


def test_census_pins(tq):
    """test_pipeline.cpp:169-190 and the BASELINE configs."""
    cfg = tq.ReconstructionConfig()
    assert tq.census(32, 32, cfg, 32) == dict(blocks=256, classes_total=81, classes_interior=64)
    cfg16 = tq.ReconstructionConfig(window=16)
    c = tq.census(32, 32, cfg16, 32)
    assert (c["classes_total"], c["classes_interior"]) == (100, 64)
    assert tq.census(512, 512, cfg, 8)["classes_total"] == 9
    assert tq.census(512, 512, cfg, 4)["classes_total"] == 4
    assert tq.census(512, 512, cfg, 16)["classes_total"] == 25
    assert tq.census(512, 512, cfg, 32)["classes_total"] == 81
    c4k = tq.census(1080, 1920, cfg, 8)
    assert c4k["blocks"] == 518400 and c4k["classes_total"] == 9
    assert tq.census(1080, 1920, cfg, 32)["classes_total"] == 90


def test_census_matches_oracle_random_shapes(tq, orc):
    rng = np.random.default_rng(0)
    for _ in range(20):
        W = int(rng.choice([8, 16, 32]))
        B = int(rng.choice([2, 4]))
        P = int(rng.choice([8, 16, 32]))
        fr, fc = int(rng.integers(W // 2, 90)), int(rng.integers(W // 2, 90))
        cfg = tq.ReconstructionConfig(window=W, block=B)
        assert tq.census(fr, fc, cfg, P) == orc.census(fr, fc, W, B, P)


@pytest.mark.parametrize("changes,msg", [
    (dict(window=7), "window size must be even"),
    (dict(block=3), "block size must divide the window"),
    (dict(window=6, block=3), "center the target block"),
    (dict(max_iterations=-1), "iteration count must be non-negative"),
    (dict(step_width=0.0), "step width must lie in (0,1]"),
    (dict(step_width=1.5), "step width must lie in (0,1]"),
    (dict(threads=-2), "thread count must be non-negative"),
])
def test_validation_messages(tq, changes, msg):
    """test_pipeline.cpp:105-147 (configuration validation)."""
    cfg = tq.ReconstructionConfig(window=16, max_iterations=30, clip_output=False)
    for k, v in changes.items():
        setattr(cfg, k, v)
    with pytest.raises(ValueError, match=re.escape(msg)):
        tq.validate_config(cfg, 32)


def test_validation_period_and_size(tq):
    cfg = tq.ReconstructionConfig(window=16)
    with pytest.raises(ValueError, match="divide the pattern period"):
        tq.validate_config(cfg, 6)
    with pytest.raises(ValueError, match="smaller than the model window"):
        tq.census(8, 8, tq.ReconstructionConfig(window=32), 32)
    with pytest.raises(ValueError, match="empty measurement frame"):
        tq.census(0, 0, cfg, 32)


def test_no_cpu_fallback(tq):
    if tq.device_count() > 0:
        pytest.skip("a CUDA device is present")
    pat = tq.generate_pattern(7, 8)
    with pytest.raises(tq.NoDeviceError):
        tq.Plan(pat, tq.ReconstructionConfig())
    frame = np.zeros((32, 32))
    with pytest.raises(tq.NoDeviceError):
        tq.reconstruct(frame, pat, tq.ReconstructionConfig())


def test_psnr(tq):
    a, b = np.zeros((4, 4)), np.ones((4, 4))
    assert tq.psnr(a, b) == 0.0
    assert tq.psnr(a, a) == float("inf")
    with pytest.raises(ValueError):
        tq.psnr(a, np.zeros((4, 5)))


def test_pad_to_block_multiple(tq):
    """test_pipeline.cpp:35-70."""
    img = tq.synthetic_image(9, 10, 1)
    padded, r, c = tq.pad_to_block_multiple(img, 4)
    assert padded.shape == (12, 12) and (r, c) == (9, 10)
    np.testing.assert_array_equal(padded[:9, :10], img)
    np.testing.assert_array_equal(padded[9:, :10], np.repeat(img[8:9], 3, 0))
    assert tq.pad_to_block_multiple(img, 3)[0].shape == (12, 12)


def test_output_buffers_are_validated():
    """Caller-supplied outputs go straight to the kernels / staging copies: wrong dtype,
    shape, layout or count must be rejected before any C call (no device needed)."""
    import numpy as np
    import paper_2205_02646_b200 as tq
    ok = np.empty((4, 6))
    assert tq._out_array(ok, (4, 6)) is ok
    assert tq._out_array(None, (4, 6)).shape == (4, 6)
    for bad in (np.empty((4, 6), np.float32), np.empty((4, 5)), np.empty((6, 4)).T,
                np.empty((4, 12))[:, ::2], [[0.0] * 6] * 4):
        with pytest.raises(ValueError):
            tq._out_array(bad, (4, 6))
    ro = np.empty((4, 6))
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        tq._out_array(ro, (4, 6))


def test_per_call_entry_points_reject_null_arguments(tq):
    """The *_with entry points (per-call config over a shared plan) fail cleanly on a
    null plan or buffer, with EINVAL (std::invalid_argument) -- no device needed."""
    import ctypes as C
    cfg = tq.ReconstructionConfig()._c()
    buf = np.zeros(16)
    rep = tq._Report()
    for rc in (tq.lib.tqsb_reconstruct_with(None, C.byref(cfg), tq._d(buf), 2, 2, tq._d(buf), None,
                                            C.byref(rep)),
               tq.lib.tqsb_reconstruct_band_with(None, C.byref(cfg), tq._d(buf), 2, 2, 0, 1,
                                                 tq._d(buf), C.byref(rep)),
               tq.lib.tqsb_reconstruct_batch_with(None, C.byref(cfg), None, 1, 2, 2, None,
                                                  C.byref(rep)),
               tq.lib.tqsb_reconstruct_device_with(None, C.byref(cfg), None, 2, 2, None, None,
                                                   C.byref(rep))):
        assert rc == tq.TQSB_EINVAL
    assert "null" in tq.lib.tqsb_last_error().decode()


def test_report_struct_matches_header(tq):
    """tqsb_report gained `compute` (the arithmetic a call ran in): the ctypes mirror and
    the header agree on the field order."""
    import os
    import re as _re
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "include", "tqsb", "tqsb.h")).read()
    body = hdr[hdr.index("typedef struct tqsb_report {"):hdr.index("} tqsb_report;")]
    fields = _re.findall(r"^\s+(?:double|long long|int)\s+(\w+);", body, _re.M)
    assert fields == [f for f, _ in tq._Report._fields_]


def test_config_struct_matches_header(tq):
    import os
    import re as _re
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "include", "tqsb", "tqsb.h")).read()
    body = hdr[hdr.index("typedef struct tqsb_config {"):hdr.index("} tqsb_config;")]
    fields = _re.findall(r"^\s+(?:double|int)\s+(\w+);", body, _re.M)
    assert fields == [f for f, _ in tq._Config._fields_]
