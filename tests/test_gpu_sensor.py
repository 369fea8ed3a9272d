"""Input side on the device: the sensor readout
(simulate_measurement, grid.cpp:46-66) bitwise equal to the host/reference one, the
synthetic scene within a few ulp of the host generator, and a scene -> readout ->
reconstruction stream that never touches the host."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,cols,period", [(64, 64, 8), (48, 80, 16), (128, 96, 32), (34, 50, 6)])
def test_device_readout_bitwise(tq, ref, need_gpu, rows, cols, period):
    import torch
    img = tq.synthetic_image(rows, cols, rows + cols)
    pat = tq.generate_pattern(3, period, 2 if period % 4 else 4)
    want = ref.simulate(img, pat.opaque, period)
    d_img = torch.from_numpy(img).cuda()
    d_frame = torch.empty((rows // 2, cols // 2), dtype=torch.float64, device="cuda")
    cfg = tq.ReconstructionConfig(window=8, block=2)
    with tq.Plan(pat, cfg) as plan:
        plan.simulate_device(d_img.data_ptr(), rows, cols, d_frame.data_ptr(),
                             torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    assert d_frame.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("rows,cols,seed", [(128, 128, 301), (1024, 1024, 1000), (270, 480, 501)])
def test_device_scene_matches_host(tq, need_gpu, rows, cols, seed):
    import torch
    d = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
    tq.synthetic_image_device(rows, cols, seed, d.data_ptr())
    torch.cuda.synchronize()
    host = tq.synthetic_image(rows, cols, seed)
    assert np.abs(d.cpu().numpy() - host).max() <= 1e-12


def test_sensor_in_the_loop_stream(tq, need_gpu):
    """scene -> readout -> reconstruction on the device for 4 frames; outputs agree
    with the host-input path within the product tolerance."""
    import torch
    rows = cols = 256
    pat = tq.generate_pattern(7, 16)
    cfg = tq.ReconstructionConfig(clip_output=False)
    s = torch.cuda.current_stream().cuda_stream
    d_img = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
    d_frame = torch.empty((rows // 2, cols // 2), dtype=torch.float64, device="cuda")
    d_out = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
    with tq.Plan(pat, cfg) as plan:
        plan.warm(rows // 2, cols // 2)
        for i in range(4):
            tq.synthetic_image_device(rows, cols, 1000 + i, d_img.data_ptr(), stream=s)
            plan.simulate_device(d_img.data_ptr(), rows, cols, d_frame.data_ptr(), s)
            plan.reconstruct_device(d_frame.data_ptr(), rows // 2, cols // 2, d_out.data_ptr(), s)
            torch.cuda.synchronize()
            gt = tq.synthetic_image(rows, cols, 1000 + i)
            host = plan.reconstruct(tq.simulate_measurement(gt, pat)).output
            out = d_out.cpu().numpy()
            assert np.abs(out - host).max() <= 1e-2
            assert abs(tq.psnr(gt, out) - tq.psnr(gt, host)) <= 0.01
