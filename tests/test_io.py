"""File formats against the unmodified reference's io.cpp:
byte-identical writers, readers that accept and reject exactly what the reference
does (with the same messages), and the known-answer cases of the reference's own
tests/test_io.cpp. CPU only."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def both_write(tq, ref, tmp_path, name, ours, theirs):
    a, b = str(tmp_path / ("ours_" + name)), str(tmp_path / ("ref_" + name))
    ours(a)
    theirs(b)
    return open(a, "rb").read(), open(b, "rb").read(), a, b


@pytest.mark.parametrize("shape,seed", [((12, 9), 3), ((64, 64), 8), ((1, 3), 1), ((33, 38), 11)])
@pytest.mark.parametrize("bits", [8, 16])
def test_pgm_bytes_identical(tq, ref, tmp_path, shape, seed, bits):
    img = tq.synthetic_image(*shape, seed) if min(shape) > 1 else np.array([[0.0, 1.0, 258 / 65535]])
    img = img.copy()
    img.flat[0] = -0.25  # clamping
    img.flat[-1] = 1.75
    a, b, pa, pb = both_write(tq, ref, tmp_path, "x.pgm", lambda p: tq.write_pgm(p, img, bits),
                              lambda p: ref.write_pgm(p, img, bits))
    assert a == b
    np.testing.assert_array_equal(tq.read_pgm(pa), ref.read(pb, 1))


def test_pgm_known_answers(tq, tmp_path):
    """test_io.cpp:47-103: exact 8-bit levels, half-step 16-bit error, big-endian samples."""
    img = np.array([[((r * 5 + c) * 17 % 256) / 255.0 for c in range(5)] for r in range(3)])
    p = str(tmp_path / "a.pgm")
    tq.write_pgm(p, img, 8)
    np.testing.assert_array_equal(tq.read_pgm(p), img)
    img16 = tq.synthetic_image(12, 9, 3)
    tq.write_pgm(p, img16, 16)
    assert np.abs(tq.read_pgm(p) - img16).max() <= 0.5 / 65535 + 1e-12
    tq.write_pgm(p, np.array([[0.0, 1.0, 258.0 / 65535.0]]), 16)
    assert open(p, "rb").read()[-6:] == bytes([0, 0, 0xFF, 0xFF, 0x01, 0x02])
    tq.write_pgm(p, np.array([[-0.25, 1.75]]), 16)
    np.testing.assert_array_equal(tq.read_pgm(p), [[0.0, 1.0]])


PGM_CASES = [
    b"P5 # magic\n# a comment line\n  2\t1 # dims\n255\n\x00\xff",  # comments, odd whitespace
    b"P2\n2 2\n255\n0 0 0 0\n",
    b"P5\n2 2\n255\nab",  # truncated
    b"P5\n0 2\n255\n",
    b"P5\n2 2\n0\n",
    b"P5\n2 2\n70000\n",
    b"P5\n2 x\n255\n",
    b"P5\n2 2\n256\n" + bytes(8),  # 16-bit samples
    b"P5\n2 2\n255\n" + bytes(4) + b"trailing",
    b"P5\n2 2 255\n\x01\x02\x03\x04",
    b"P5\n2 2\n255",  # header ends at EOF
    b"P5\n2#c\n2\n255\n1234",
    b"",
    b"P5\n-2 2\n255\n",
    b"P5\n2 2\n+255\n1234",
]


@pytest.mark.parametrize("content", PGM_CASES)
def test_pgm_reader_accepts_and_rejects_like_reference(tq, ref, tmp_path, content):
    p = str(tmp_path / "f.pgm")
    open(p, "wb").write(content)
    want = got = None
    try:
        want = ref.read(p, 1)
    except RuntimeError as e:
        want = ("error", str(e))
    try:
        got = tq.read_pgm(p)
    except tq.FormatError as e:
        got = ("error", str(e))
    if isinstance(want, tuple):
        assert got == want
    else:
        np.testing.assert_array_equal(got, want)


def test_pgm_write_validation(tq, ref, tmp_path):
    """test_io.cpp:130-133: bit depth 8|16 and non-empty images are invalid_argument."""
    p = str(tmp_path / "g.pgm")
    with pytest.raises(ValueError, match="bit depth must be 8 or 16"):
        tq.write_pgm(p, np.zeros((2, 2)), 12)
    with pytest.raises(ValueError, match="empty image"):
        tq.write_pgm(p, np.zeros((0, 0)), 8)
    with pytest.raises(tq.FormatError, match="missing.pgm: cannot open for reading"):
        tq.read_pgm(str(tmp_path / "missing.pgm"))


@pytest.mark.parametrize("seed,period", [(7, 32), (7, 8), (3, 16), (2**63 + 5, 4), (0, 64)])
def test_pattern_files_identical_and_round_trip(tq, ref, tmp_path, seed, period):
    pat = tq.generate_pattern(seed, period, 2 if period % 4 else 4)
    a, b, pa, pb = both_write(
        tq, ref, tmp_path, "p.tqsp", lambda p: tq.write_pattern(p, pat),
        lambda p: ref.write_pattern(p, period, seed, "mt19937_64", pat.opaque))
    assert a == b
    back = tq.read_pattern(pa)
    assert (back.period, back.seed, back.rng) == (period, seed, "mt19937_64")
    np.testing.assert_array_equal(back.opaque, pat.opaque)
    if (seed, period) == (7, 32):
        assert a.split(b"\n")[0] == b"TQSP v1 period=32 seed=7 rng=mt19937_64"


PATTERN_CASES = [
    "TQSQ v1 period=4 seed=1 rng=x\n0 1\n2 3\n",
    "TQSP v2 period=4 seed=1 rng=x\n0 1\n2 3\n",
    "TQSP v1 period=4 rng=x\n0 1\n2 3\n",
    "TQSP v1 period=5 seed=1 rng=x\n0 1\n2 3\n",
    "TQSP v1 period=4 seed=1 rng=x\n0 7\n2 3\n",
    "TQSP v1 period=4 seed=1 rng=x\n0 1 2\n2 3\n",
    "TQSP v1 period=4 seed=1 rng=x\n0 1\n",
    "TQSP v1 period=4 seed=1 rng=x bogus=3\n0 1\n2 3\n",
    "TQSP v1 period=4 seed=1 rng=x\n0 1\n2 3\n",
    "TQSP v1 period=4 seed=1\n0 1\n2 3\n",
    "TQSP v1 period=4 seed=-1 rng=x\n01 1\n2 3\n",
    "TQSP v1 period=4 seed=12ab rng=x\n0 1\n2 3 \n",
    "TQSP v1 period=4 seed=x rng=x\n0 1\n2 3\n",
    "TQSP v1 period=4x seed=1 rng=x\n0 1\n2 3\n",
    "TQSP v1 period seed=1\n0 1\n2 3\n",
    "",
    "TQSP v1 period=2 seed=1 rng=x\n0\n",
]


@pytest.mark.parametrize("content", PATTERN_CASES)
def test_pattern_reader_like_reference(tq, ref, tmp_path, content):
    """test_io.cpp:161-189 plus edge cases; outcomes and messages must agree."""
    p = str(tmp_path / "p.tqsp")
    open(p, "w").write(content)
    try:
        want = ref.read_pattern(p)
    except (RuntimeError, ValueError) as e:
        want = ("error", str(e))
    try:
        got = tq.read_pattern(p)
        got = (got.period, got.seed, got.rng, got.opaque)
    except tq.FormatError as e:
        got = ("error", str(e))
    if want[0] == "error":
        assert got == want
    else:
        assert got[:3] == want[:3]
        np.testing.assert_array_equal(got[3], want[3])


def test_tqsm_identical_and_bitwise(tq, ref, tmp_path):
    """test_io.cpp:192-232: frames and raw dumps round trip bitwise; read_image_any sniffs."""
    rng = np.random.default_rng(19)
    f = rng.uniform(-2, 2, (3, 7))
    f[0, 4] = 0.1 + 0.2
    f[1, 1] = -0.0
    f[2, 2] = np.inf
    a, b, pa, pb = both_write(tq, ref, tmp_path, "y.tqsm", lambda p: tq.write_frame(p, f),
                              lambda p: ref.write_tqsm(p, f))
    assert a == b
    back = tq.read_frame(pa)
    assert back.tobytes() == f.tobytes()
    img = tq.synthetic_image(10, 14, 77)
    tq.write_raw_image(pa, img)
    assert tq.read_image_any(pa).tobytes() == img.tobytes()
    tq.write_pgm(pb, img, 16)
    assert np.abs(tq.read_image_any(pb) - img).max() <= 0.5 / 65535 + 1e-12


def test_tqsm_rejects_like_reference(tq, ref, tmp_path):
    p = str(tmp_path / "z.tqsm")
    f = np.full((2, 2), 0.5)
    tq.write_frame(p, f)
    good = open(p, "rb").read()
    cases = [b"NOPE####", b"TQSM" + b"\xff" * 8, good[:-9], b"TQSM\x01\x00", b"TQS",
             b"TQSM" + bytes(8), good + b"extra"]
    for c in cases:
        open(p, "wb").write(c)
        try:
            want = ref.read(p, 2)
        except RuntimeError as e:
            want = ("error", str(e))
        try:
            got = tq.read_frame(p)
        except tq.FormatError as e:
            got = ("error", str(e))
        if isinstance(want, tuple):
            assert got == want, c
        else:
            np.testing.assert_array_equal(got, want)
    with pytest.raises(tq.FormatError, match="missing.tqsm"):
        tq.read_frame(str(tmp_path / "missing.tqsm"))


def test_cross_reading(tq, ref, tmp_path):
    """Files written by the reference read bitwise identically here and vice versa."""
    img = tq.synthetic_image(40, 24, 5)
    for bits in (8, 16):
        ref.write_pgm(str(tmp_path / "r.pgm"), img, bits)
        tq.write_pgm(str(tmp_path / "o.pgm"), img, bits)
        np.testing.assert_array_equal(tq.read_image_any(str(tmp_path / "r.pgm")),
                                      ref.read(str(tmp_path / "o.pgm"), 0))
    ref.write_tqsm(str(tmp_path / "r.tqsm"), img)
    assert tq.read_image_any(str(tmp_path / "r.tqsm")).tobytes() == img.tobytes()
