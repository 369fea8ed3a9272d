"""TQSK table persistence (rljsde.cpp:322-475): pattern digest
and memory accounting pinned against the reference (CPU), and on the GPU the file
round trip, interchange with the reference's save_kernel_cache / load_kernel_cache
in both directions, and header validation."""
import os

import numpy as np
import pytest


@pytest.mark.parametrize("seed,period", [(7, 32), (1, 4), (99, 16), (3, 64), (7, 8), (0, 6)])
def test_pattern_digest_matches_reference(tq, ref, seed, period):
    p = tq.generate_pattern(seed, period, 2 if period % 4 else 4)
    assert tq.pattern_digest(p) == ref.pattern_digest(p.opaque, period)


@pytest.mark.parametrize("classes,window,double,local", [
    (64, 32, False, -1), (64, 32, True, -1), (0, 16, True, -1), (9, 32, True, 256), (81, 8, False, 3)])
def test_memory_report_matches_reference(tq, ref, classes, window, double, local):
    prec = tq.PRECISION_DOUBLE if double else tq.PRECISION_SINGLE
    assert tq.kernel_memory_report(classes, window, prec, local) == \
        ref.memory_report(classes, window, double, local)


def test_memory_report_known_answers(tq):
    """test_cli.cpp:271-293: 64 classes, W = 32, single -> 671,612,928 bytes; double 2x."""
    r = tq.kernel_memory_report(64, 32, tq.PRECISION_SINGLE)
    assert (r["b_bytes"], r["c_bytes"], r["d_bytes"], r["total_bytes"]) == \
        (134217728, 536870912, 524288, 671612928)
    assert tq.kernel_memory_report(64, 32, tq.PRECISION_DOUBLE)["total_bytes"] == 2 * 671612928
    with pytest.raises(ValueError):
        tq.kernel_memory_report(-3, 32)


def _setup(tq, rows=48, cols=48, seed=61, period=32):
    gt = tq.synthetic_image(rows, cols, seed)
    pat = tq.generate_pattern(7, period)
    return gt, pat, tq.simulate_measurement(gt, pat)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["double", "single"])
def test_tqsk_round_trip_skips_precompute(tq, need_gpu, tmp_path, precision):
    gt, pat, frame = _setup(tq)
    prec = tq.PRECISION_DOUBLE if precision == "double" else tq.PRECISION_SINGLE
    cfg = tq.ReconstructionConfig(window=16, max_iterations=6, precision=prec)
    path = str(tmp_path / "k.tqsk")
    with tq.Plan(pat, cfg) as plan:
        first = plan.reconstruct(frame)
        assert first.classes_created > 0
        n = plan.save_tables(path)
        assert n == plan.stats()["classes"]
    with tq.Plan(pat, cfg) as plan2:
        assert plan2.load_tables(path) == n
        second = plan2.reconstruct(frame)
        assert second.classes_created == 0
        if precision == "double":  # fp64 planes round trip exactly
            np.testing.assert_array_equal(second.output, first.output)
        else:  # planes stored as fp32: the product path tolerance
            assert np.abs(second.output - first.output).max() <= 1e-2
            assert abs(tq.psnr(gt, second.output) - tq.psnr(gt, first.output)) <= 0.01
        # the same file saved again is byte-identical
        plan2.save_tables(str(tmp_path / "k2.tqsk"))
    assert open(path, "rb").read() == open(str(tmp_path / "k2.tqsk"), "rb").read()


@pytest.mark.gpu
def test_tqsk_header_mismatch_is_rejected(tq, need_gpu, tmp_path):
    gt, pat, frame = _setup(tq)
    cfg = tq.ReconstructionConfig(window=16, max_iterations=6)
    path = str(tmp_path / "k.tqsk")
    with tq.Plan(pat, cfg) as plan:
        plan.reconstruct(frame)
        plan.save_tables(path)
    for other in [tq.ReconstructionConfig(window=16, precision=tq.PRECISION_SINGLE),
                  tq.ReconstructionConfig(window=16, spatial_decay=0.7),
                  tq.ReconstructionConfig(window=32)]:
        with tq.Plan(pat, other) as p2, pytest.raises(tq.FormatError, match="does not match"):
            p2.load_tables(path)
    with tq.Plan(tq.generate_pattern(8, 32), cfg) as p3, pytest.raises(tq.FormatError):
        p3.load_tables(path)
    open(str(tmp_path / "bad.tqsk"), "wb").write(b"NOPE")
    with tq.Plan(pat, cfg) as p4:
        with pytest.raises(tq.FormatError, match="not a TQSK kernel cache"):
            p4.load_tables(str(tmp_path / "bad.tqsk"))
        raw = open(path, "rb").read()
        open(str(tmp_path / "trunc.tqsk"), "wb").write(raw[: len(raw) // 2])
        with pytest.raises(tq.FormatError, match="truncated class payload"):
            p4.load_tables(str(tmp_path / "trunc.tqsk"))


@pytest.mark.gpu
def test_tqsk_interchange_with_reference(tq, ref, need_gpu, tmp_path):
    """A reference-written cache drives our plan and ours drives the reference."""
    gt, pat, frame = _setup(tq, 64, 64, 301, 8)
    W, it = 32, 30
    cfg64 = tq.ReconstructionConfig(window=W, max_iterations=it, clip_output=False,
                                     compute=tq.COMPUTE_FP64)
    want, _ = ref.reconstruct(frame, pat.opaque, 8, window=W, iterations=it, clip=False)
    # reference -> ours
    rc = ref.new_cache()
    try:
        ref.reconstruct(frame, pat.opaque, 8, window=W, iterations=it, clip=False, cache=rc)
        ref.save_cache(rc, str(tmp_path / "ref.tqsk"), pat.opaque, 8, W)
    finally:
        ref.free_cache(rc)
    with tq.Plan(pat, cfg64) as plan:
        assert plan.load_tables(str(tmp_path / "ref.tqsk")) > 0
        rep = plan.reconstruct(frame)
        assert rep.classes_created == 0
        assert np.abs(rep.output - want).max() <= 1e-9
        plan.save_tables(str(tmp_path / "ours.tqsk"))
    # ours -> reference
    rc = ref.new_cache()
    try:
        n = ref.load_cache(rc, str(tmp_path / "ours.tqsk"), pat.opaque, 8, W)
        assert n > 0
        got, rrep = ref.reconstruct(frame, pat.opaque, 8, window=W, iterations=it, clip=False,
                                    cache=rc)
        assert rrep.classes_created == 0
        assert np.abs(got - want).max() <= 1e-9
    finally:
        ref.free_cache(rc)
    # the files agree in layout and size; planes to the table tolerance
    a, b = open(str(tmp_path / "ref.tqsk"), "rb").read(), open(str(tmp_path / "ours.tqsk"), "rb").read()
    assert len(a) == len(b) and a[:44] == b[:44]
