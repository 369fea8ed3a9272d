"""Profiling driver: a few device-resident reconstructions of one workload
(default 1 MP, P = 8, reference defaults) so ncu can capture k_solve_f32."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_02646_b200 as tq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=1024)
ap.add_argument("--cols", type=int, default=1024)
ap.add_argument("--period", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--hot", type=int, default=-1)
a = ap.parse_args()
gt = tq.synthetic_image(a.rows, a.cols, 401)
pat = tq.generate_pattern(7, a.period)
frame = tq.simulate_measurement(gt, pat)
plan = tq.Plan(pat, tq.ReconstructionConfig(hot_columns=a.hot))
plan.warm(*frame.shape)
d_frame = torch.from_numpy(frame).cuda()
d_out = torch.empty((a.rows, a.cols), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
for i in range(a.reps):
    ev[2 * i].record(s)
    plan.reconstruct_device(d_frame.data_ptr(), frame.shape[0], frame.shape[1], d_out.data_ptr(),
                            s.cuda_stream)
    ev[2 * i + 1].record(s)
torch.cuda.synchronize()
print("ms:", [round(ev[2 * i].elapsed_time(ev[2 * i + 1]), 3) for i in range(a.reps)])
