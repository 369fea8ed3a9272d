"""Per-phase cycle accounting of the solve loop from a TQSB_TIMING=1 build:
  python paper_2205_02646_b200/build.py timing TQSB_ONLY_W32 TQSB_TIMING=1
  TQSB_LIB=.../libtqsb_timing.so python tools/chain_timing.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_02646_b200 as tq  # noqa: E402

rows, cols = 2160, 3840
gt = tq.synthetic_image(rows, cols, 501)
pat = tq.generate_pattern(7, 8)
frame = tq.simulate_measurement(gt, pat)
plan = tq.Plan(pat, tq.ReconstructionConfig())
plan.warm(*frame.shape)
d_frame = torch.from_numpy(frame).cuda()
d_out = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
plan.reconstruct_device(d_frame.data_ptr(), frame.shape[0], frame.shape[1], d_out.data_ptr(), 0)
torch.cuda.synchronize()
out = (C.c_ulonglong * 6)()
tq.lib.tqsb_debug_timing(out)
n_tm, n_g = out[4], out[5]
n = n_tm + n_g
print(f"iterations {n}  tmem {n_tm / n:.3f}  global {n_g / n:.3f}")
print(f"argmax->u        {out[0] / n:8.1f} cycles")
print(f"u->g ready       {out[1] / n:8.1f} cycles")
print(f"update (tmem)    {out[2] / max(n_tm, 1):8.1f} cycles")
print(f"update (global)  {out[3] / max(n_g, 1):8.1f} cycles")
print(f"per iteration    {(out[0] + out[1] + out[2] + out[3]) / n:8.1f} cycles (one warp, 3 share an SMSP)")
