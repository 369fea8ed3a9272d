"""Where does the e2e time go? Host-buffer band runs with pinned buffers."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_02646_b200 as tq  # noqa: E402

gt = tq.synthetic_image(2160, 3840, 501)
pat = tq.generate_pattern(7, 8)
frame = tq.simulate_measurement(gt, pat)
fr, fc = frame.shape
plan = tq.Plan(pat, tq.ReconstructionConfig())
hin = tq.lib.tqsb_host_alloc(frame.nbytes)
hout = tq.lib.tqsb_host_alloc(4 * frame.nbytes)
h_in = np.ctypeslib.as_array((ctypes.c_double * frame.size).from_address(hin)).reshape(frame.shape)
h_out = np.ctypeslib.as_array((ctypes.c_double * (4 * frame.size)).from_address(hout)).reshape(2 * fr, 2 * fc)
h_in[...] = frame
for i in range(6):
    t = time.perf_counter()
    rep = plan.reconstruct_band(h_in, 0, 540, out=h_out)
    w = time.perf_counter() - t
    print(f"wall {w*1e3:.2f} ms  lib e2e {rep.e2e_seconds*1e3:.2f}  kernels {rep.seconds*1e3:.2f} launches {rep.gpu_launches}")
for i in range(3):
    t = time.perf_counter()
    rep = plan.reconstruct(frame)
    w = time.perf_counter() - t
    print(f"pageable full: wall {w*1e3:.2f} ms  lib e2e {rep.e2e_seconds*1e3:.2f}  kernels {rep.seconds*1e3:.2f}")
