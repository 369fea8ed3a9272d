"""Fixed (init + placement) vs per-iteration cost of the solve kernel at 4K:
device time of one frame at nu = 0, 1, 50, 200 iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_02646_b200 as tq  # noqa: E402

rows, cols = 2160, 3840
gt = tq.synthetic_image(rows, cols, 501)
pat = tq.generate_pattern(7, 8)
frame = tq.simulate_measurement(gt, pat)
d_frame = torch.from_numpy(frame).cuda()
d_out = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
for nu in (0, 1, 50, 200):
    plan = tq.Plan(pat, tq.ReconstructionConfig(max_iterations=nu))
    plan.warm(*frame.shape)
    ms = []
    for i in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.reconstruct_device(d_frame.data_ptr(), *frame.shape, d_out.data_ptr(), 0)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    print(f"nu={nu:4d}  {min(ms[1:]):8.3f} ms")
    plan.close()
