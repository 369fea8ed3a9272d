"""The `tqsb` command-line toolbox -- the reference's `tqs`
tool (tools/tqs.cpp) with its flags, report keys and exit codes. The cases follow
the reference's tests/test_cli.cpp; outputs are checked against the unmodified
reference library (file bytes, frames). Subcommands that reconstruct need a GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2205_02646_b200", "bin", "tqsb")


def run(*args):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


@pytest.fixture(scope="module", autouse=True)
def cli_built(tq):
    if not os.path.exists(CLI):
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "b", os.path.join(ROOT, "paper_2205_02646_b200", "build.py"))
        m = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(m)
        m.build_cli()
    assert os.path.exists(CLI)


def test_pattern_subcommand_deterministic_and_validated(tq, ref, tmp_path):
    a, b = tmp_path / "a.tqsp", tmp_path / "b.tqsp"
    rc, out, _ = run("pattern", "--seed", 7, "--period", 32, "-o", a)
    assert rc == 0 and "period=32" in out
    assert run("pattern", "--seed", 7, "--period", 32, "-o", b)[0] == 0
    assert a.read_bytes() == b.read_bytes()
    # byte-identical to the reference's write_pattern
    ref.write_pattern(str(tmp_path / "r.tqsp"), 32, 7, "mt19937_64", ref.generate_pattern(7, 32))
    assert a.read_bytes() == (tmp_path / "r.tqsp").read_bytes()
    p = tq.read_pattern(str(a))
    assert p.seed == 7
    np.testing.assert_array_equal(p.opaque, ref.generate_pattern(7, 32))
    assert run("pattern", "--seed", 1, "--period", 30, "-o", tmp_path / "x.tqsp")[0] == 2
    assert run("pattern", "--seed", 1, "--period", 32)[0] == 2
    assert run("pattern", "--seed=7", "--period=16", "--output", tmp_path / "c.tqsp")[0] == 0
    assert tq.read_pattern(str(tmp_path / "c.tqsp")).period == 16


def test_top_level_usage(tmp_path):
    assert run()[0] == 2
    assert run("frobnicate")[0] == 2
    assert run("--help")[0] == 0
    rc, out, _ = run("reconstruct", "--help")
    assert rc == 0 and "--kernel-cache" in out
    assert run("pattern", "--bogus", 1, "-o", tmp_path / "p")[0] == 2
    assert run("pattern", "--period", "abc", "-o", tmp_path / "p")[0] == 2


def test_simulate_produces_reference_frame(tq, ref, tmp_path):
    run("pattern", "--seed", 3, "--period", 16, "-o", tmp_path / "p.tqsp")
    img = tq.synthetic_image(32, 48, 55)
    tq.write_raw_image(str(tmp_path / "in.tqsm"), img)
    rc, out, _ = run("simulate", "--image", tmp_path / "in.tqsm", "--pattern", tmp_path / "p.tqsp",
                     "-o", tmp_path / "y.tqsm")
    assert rc == 0 and "16x24 frame" in out
    got = tq.read_frame(str(tmp_path / "y.tqsm"))
    want = ref.simulate(img, ref.generate_pattern(3, 16), 16)
    assert got.tobytes() == want.tobytes()
    rc, _, err = run("simulate", "--image", tmp_path / "nope.tqsm", "--pattern",
                     tmp_path / "p.tqsp", "-o", tmp_path / "z.tqsm")
    assert rc == 2 and "error:" in err


def test_compare_gates_on_threshold(tq, tmp_path):
    img = tq.synthetic_image(24, 24, 70)
    tq.write_raw_image(str(tmp_path / "a.tqsm"), img)
    pert = img.copy()
    pert[3, 4] += 0.125
    tq.write_raw_image(str(tmp_path / "b.tqsm"), pert)
    rc, out, _ = run("compare", tmp_path / "a.tqsm", tmp_path / "a.tqsm", "--threshold", 0)
    assert rc == 0 and "PASS" in out
    rc, out, _ = run("compare", tmp_path / "a.tqsm", tmp_path / "b.tqsm")
    assert rc == 1 and "FAIL" in out
    rc, out, _ = run("compare", tmp_path / "a.tqsm", tmp_path / "b.tqsm", "--threshold", 0.2,
                     "--reference", tmp_path / "a.tqsm", "--format", "json")
    assert rc == 0
    j = json.loads(out)
    assert j["pass"] is True
    assert j["max_abs_diff"] == pytest.approx(0.125, rel=1e-12)
    assert j["psnr_a_vs_ref"] == "identical"
    assert isinstance(j["psnr_b_vs_ref"], float)
    assert list(j) == sorted(j)  # nlohmann's std::map key order
    assert '"threshold": 0.2\n' in out and '"pass": true,' in out
    tq.write_raw_image(str(tmp_path / "c.tqsm"), np.full((8, 8), 0.5))
    assert run("compare", tmp_path / "a.tqsm", tmp_path / "c.tqsm")[0] == 2


def test_kernel_report(tq):
    rc, out, _ = run("kernel-report", "--classes", 64, "--window", 32, "--precision", "single")
    assert rc == 0
    for s in ["134.217728", "536.870912", "0.524288", "671.612928"]:
        assert s in out
    rc, out, _ = run("kernel-report", "--classes", 64, "--window", 32, "--precision", "single",
                     "--format", "json")
    j = json.loads(out)
    assert (j["b_bytes"], j["c_bytes"], j["d_bytes"], j["total_bytes"]) == \
        (134217728, 536870912, 524288, 671612928)
    assert '"b_mb": 134.217728,' in out
    rc, out, _ = run("kernel-report", "--classes", 64, "--window", 32, "--precision", "double",
                     "--format", "json")
    assert json.loads(out)["total_bytes"] == 2 * 671612928
    assert run("kernel-report", "--classes", -3)[0] == 2
    assert run("kernel-report", "--precision", "half")[0] == 2


# ---------------------------------------------------------------- GPU subcommands
def _recon_setup(tq, tmp_path, seed=60):
    run("pattern", "--seed", 7, "--period", 32, "-o", tmp_path / "p.tqsp")
    img = tq.synthetic_image(48, 48, seed)
    tq.write_raw_image(str(tmp_path / "ref.tqsm"), img)
    tq.write_frame(str(tmp_path / "y.tqsm"),
                   tq.simulate_measurement(img, tq.generate_pattern(7, 32)))
    return img, ["reconstruct", "--input", tmp_path / "y.tqsm", "--pattern", tmp_path / "p.tqsp",
                 "--window", 16, "--iterations", 8, "--threads", 1]


@pytest.mark.gpu
def test_reconstruct_reports_and_images(tq, ref, need_gpu, tmp_path):
    img, base = _recon_setup(tq, tmp_path)
    rc, out, err = run(*base, "-o", tmp_path / "out.pgm", "--reference", tmp_path / "ref.tqsm")
    assert rc == 0, err
    assert "algorithm:        rljsde" in out and "blocks:           144" in out
    assert "psnr vs ref:" in out
    o = tq.read_pgm(str(tmp_path / "out.pgm"))
    assert o.shape == (48, 48)
    rc, out, err = run(*base, "-o", tmp_path / "out.pgm", "--raw", tmp_path / "out.tqsm",
                       "--bits", 16, "--format", "json")
    assert rc == 0, err
    j = json.loads(out)
    assert (j["algorithm"], j["blocks"], j["rows"], j["cols"], j["window"]) == \
        ("rljsde", 144, 48, 48, 16)
    raw = tq.read_raw_image(str(tmp_path / "out.tqsm"))
    q = tq.read_pgm(str(tmp_path / "out.pgm"))
    assert np.abs(raw - q).max() <= 0.5 / 65535 + 1e-12
    # the raw output is the reference's reconstruction within the fp32 tolerance
    frame = tq.read_frame(str(tmp_path / "y.tqsm"))
    want, _ = ref.reconstruct(frame, tq.generate_pattern(7, 32).opaque, 32, window=16,
                              iterations=8)
    assert np.abs(raw - want).max() <= 1e-2
    rc, out, err = run(*base, "--compute", "fp64", "--raw", tmp_path / "o64.tqsm",
                       "-o", tmp_path / "o64.pgm")
    assert rc == 0, err
    assert np.abs(tq.read_raw_image(str(tmp_path / "o64.tqsm")) - want).max() <= 1e-9
    rc, out, err = run("reconstruct", "--input", tmp_path / "y.tqsm", "--pattern",
                       tmp_path / "p.tqsp", "--window", 16, "--iterations", 4, "--threads", 1,
                       "--algo", "ljsde", "-o", tmp_path / "outL.pgm", "--raw", tmp_path / "L.tqsm")
    assert rc == 0, err
    assert "algorithm:        ljsde" in out
    wantL, _ = ref.reconstruct_algo(frame, tq.generate_pattern(7, 32).opaque, 32, "ljsde",
                                    window=16, iterations=4, clip=True)
    assert np.abs(tq.read_raw_image(str(tmp_path / "L.tqsm")) - wantL).max() <= 1e-9
    assert run(*base, "--algo", "magic", "-o", tmp_path / "x.pgm")[0] == 2


@pytest.mark.gpu
def test_kernel_cache_files_short_circuit_warm_pass(tq, ref, need_gpu, tmp_path):
    img, base = _recon_setup(tq, tmp_path, 61)
    base = base[:-4] + ["--iterations", 6, "--threads", 1, "--kernel-cache", tmp_path / "k.tqsk"]
    rc, out, err = run(*base, "-o", tmp_path / "o1.pgm", "--format", "json")
    assert rc == 0, err
    assert os.path.exists(tmp_path / "k.tqsk")
    assert json.loads(out)["classes_created"] > 0
    rc, out, err = run(*base, "-o", tmp_path / "o2.pgm", "--format", "json")
    assert rc == 0, err
    assert json.loads(out)["classes_created"] == 0
    assert (tmp_path / "o1.pgm").read_bytes() == (tmp_path / "o2.pgm").read_bytes()
    rc, _, err = run(*base, "--precision", "single", "-o", tmp_path / "o3.pgm")
    assert rc == 2 and "error:" in err
    # the file is a valid reference kernel cache
    rc_ = ref.new_cache()
    try:
        assert ref.load_cache(rc_, str(tmp_path / "k.tqsk"), tq.generate_pattern(7, 32).opaque,
                              32, 16) > 0
    finally:
        ref.free_cache(rc_)


@pytest.mark.gpu
def test_bench_runs_both_algorithms(tq, need_gpu, tmp_path):
    run("pattern", "--seed", 7, "--period", 32, "-o", tmp_path / "p.tqsp")
    (tmp_path / "imgs").mkdir()
    tq.write_pgm(str(tmp_path / "imgs" / "a.pgm"), tq.synthetic_image(32, 32, 80), 16)
    tq.write_pgm(str(tmp_path / "imgs" / "b.pgm"), tq.synthetic_image(32, 32, 81), 16)
    (tmp_path / "imgs" / "ignore.txt").write_text("not an image")
    rc, out, err = run("bench", "--images", tmp_path / "imgs", "--pattern", tmp_path / "p.tqsp",
                       "--window", 16, "--iterations", 6, "--format", "json")
    assert rc == 0, err
    j = json.loads(out)
    assert j["images"] == 2
    assert j["max_abs_difference"] <= 1e-6
    assert j["speedup"] > 0.0
    assert "ljsde_scaling_ratio" not in j
    rc, out, err = run("bench", "--images", tmp_path / "imgs", "--pattern", tmp_path / "p.tqsp",
                       "--window", 32, "--iterations", 6, "--scaling", "--format", "json")
    assert rc == 0, err
    assert json.loads(out)["ljsde_scaling_ratio"] > 0.0  # tiny images: launch-bound on a GPU
    (tmp_path / "empty").mkdir()
    assert run("bench", "--images", tmp_path / "empty", "--pattern", tmp_path / "p.tqsp")[0] == 2
