"""The plan as the reference's shared KernelCache (rljsde.hpp:81-100, pipeline.cpp:108-166):
it pins the window and the fp64 tables per offset class, and every call brings its own
solver options. A cache driven with different nu, gamma, clip, frequency exponent, block
and compute must give, call by call, exactly the output of a fresh plan with that config;
L-JSDE never touches it (test_pipeline.cpp:206-216). Plus the multi-device band split
exercised on one GPU (devices = [0, 0]: two independent contexts, no kernel waits on
another) and the per-launch task-queue heads of the asynchronous device entry point."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene(tq):
    pat = tq.generate_pattern(7, 32)
    gt = tq.synthetic_image(96, 128, 12)
    return pat, gt, tq.simulate_measurement(gt, pat)


VARIANTS = [dict(max_iterations=50, step_width=1.0, clip_output=False),
            dict(max_iterations=200, step_width=0.5, clip_output=True),
            dict(max_iterations=50, step_width=0.5, frequency_exponent=1.0),
            dict(max_iterations=120, step_width=1.0, frequency_exponent=1.0, block=2),
            dict(max_iterations=60, compute=1),
            dict(max_iterations=60, compute=1, frequency_exponent=1.0, block=2, clip_output=False),
            dict(max_iterations=200, step_width=0.5, clip_output=True)]


def test_shared_cache_takes_options_per_call(tq, need_gpu, scene):
    pat, gt, frame = scene
    base = tq.ReconstructionConfig(window=16)
    with tq.Plan(pat, base) as cache:
        created = 0
        for v in VARIANTS:
            cfg = tq.ReconstructionConfig(window=16, **v)
            got = tq.reconstruct(frame, pat, cfg, cache=cache)
            with tq.Plan(pat, cfg) as fresh:
                want = fresh.reconstruct(frame)
            assert got.output.tobytes() == want.output.tobytes(), v
            assert got.compute == want.compute == (1 if v.get("compute") == 1 else 0)
            created += got.classes_created
        assert created == cache.stats()["classes"]  # the tables were built once per class
        with pytest.raises(tq.LogicError):
            tq.reconstruct(frame, pat, tq.ReconstructionConfig(window=32), cache=cache)


def test_ljsde_leaves_the_cache_untouched(tq, need_gpu, scene):
    pat, gt, frame = scene
    with tq.Plan(pat, tq.ReconstructionConfig(window=16)) as cache:
        cfg = tq.ReconstructionConfig(window=16, algorithm=tq.ALGO_LJSDE, max_iterations=2)
        rep = tq.reconstruct(frame, pat, cfg, cache=cache)
        assert cache.stats()["classes"] == 0
        assert rep.cache_hits == 0 and rep.cache_misses == 0 and rep.compute == tq.COMPUTE_FP64


def test_block_above_16_runs_on_the_fp64_kernel(tq, ref, need_gpu, scene):
    """B = 32 (W = 32): accepted by the reference (pipeline.cpp:27-42); served by the fp64
    kernel, i.e. the reference's exact greedy paths."""
    pat, gt, frame = scene
    cfg = tq.ReconstructionConfig(block=32, max_iterations=40, clip_output=False)
    rep = tq.reconstruct(frame, pat, cfg)
    assert rep.compute == tq.COMPUTE_FP64
    want, _ = ref.reconstruct(frame, pat.opaque, 32, block=32, iterations=40, clip=False)
    assert np.abs(rep.output - want).max() <= 1e-9


def test_f64r_large_nu_falls_back(tq, ref, need_gpu):
    """W = 32 with nu = 1024 in fp64 mode: the register kernel's shared layout would
    exceed 227 KB, so the launch goes to the generic kernel instead of failing."""
    pat = tq.generate_pattern(7, 8)
    gt = tq.synthetic_image(64, 64, 14)
    frame = tq.simulate_measurement(gt, pat)
    cfg = tq.ReconstructionConfig(max_iterations=1024, compute=tq.COMPUTE_FP64, clip_output=False)
    rep = tq.reconstruct(frame, pat, cfg)
    want, _ = ref.reconstruct(frame, pat.opaque, 8, iterations=1024, clip=False)
    assert np.abs(rep.output - want).max() <= 1e-9


@pytest.mark.parametrize("compute", [0, 1])
def test_two_device_contexts_on_one_gpu(tq, need_gpu, compute):
    """The in-process multi-device split (plan.cpp reconstruct_impl / batch) with
    devices = [0, 0]: bitwise equal to one device."""
    pat = tq.generate_pattern(7, 8)
    gt = tq.synthetic_image(512, 384, 15)
    frame = tq.simulate_measurement(gt, pat)
    frames = [frame, tq.simulate_measurement(tq.synthetic_image(512, 384, 16), pat), frame]
    cfg = tq.ReconstructionConfig(compute=compute, max_iterations=200 if compute == 0 else 60)
    with tq.Plan(pat, cfg, devices=[0]) as one, tq.Plan(pat, cfg, devices=[0, 0]) as two:
        a, b = one.reconstruct(frame), two.reconstruct(frame)
        assert a.output.tobytes() == b.output.tobytes()
        assert (a.blocks_processed, a.classes_total) == (b.blocks_processed, b.classes_total)
        ba, bb = one.reconstruct_batch(frames), two.reconstruct_batch(frames)
        for x, y in zip(ba.output, bb.output):
            assert x.tobytes() == y.tobytes()
        assert bb.output[0].tobytes() == a.output.tobytes()


def test_concurrent_device_launches_use_separate_queues(tq, need_gpu):
    """Two asynchronous device-resident reconstructions in flight on two streams of one
    plan: each launch has its own task-queue head, so both outputs are complete."""
    import torch
    pat = tq.generate_pattern(7, 8)
    gt = tq.synthetic_image(256, 256, 17)
    frame = tq.simulate_measurement(gt, pat)
    with tq.Plan(pat, tq.ReconstructionConfig()) as plan:
        want = plan.reconstruct(frame).output
        d_frame = torch.from_numpy(frame).cuda()
        outs = [torch.full(want.shape, -1.0, dtype=torch.float64, device="cuda") for _ in range(2)]
        streams = [torch.cuda.Stream() for _ in range(2)]
        for o, s in zip(outs, streams):
            plan.reconstruct_device(d_frame.data_ptr(), *frame.shape, o.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        for o in outs:
            assert o.cpu().numpy().tobytes() == want.tobytes()


def test_batch_mixed_pinned_and_pageable_outputs(tq, need_gpu):
    """run_batch_host: a pageable output two frames before a pinned one is still handed
    over (the staging slot is drained whatever the later frame's buffer is)."""
    import ctypes
    pat = tq.generate_pattern(7, 8)
    frames = [tq.simulate_measurement(tq.synthetic_image(128, 128, 20 + i), pat) for i in range(5)]
    with tq.Plan(pat, tq.ReconstructionConfig()) as plan:
        want = [plan.reconstruct(f).output for f in frames]
        n = 128 * 128
        ptr = tq.lib.tqsb_host_alloc(8 * n * 3)
        try:
            buf = np.ctypeslib.as_array((ctypes.c_double * (n * 3)).from_address(ptr))
            pinned = [buf[i * n:(i + 1) * n].reshape(128, 128) for i in range(3)]
            outs = [np.empty((128, 128)), np.empty((128, 128)), pinned[0], pinned[1], pinned[2]]
            plan.reconstruct_batch(frames, outs)
            for o, w in zip(outs, want):
                assert o.tobytes() == w.tobytes()
        finally:
            tq.lib.tqsb_host_free(ptr)
