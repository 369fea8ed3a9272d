"""L-JSDE baseline (ljsde.cpp) on the device vs the reference's L-JSDE on all host cores,
and both against RL-JSDE -- the paper's L vs RL comparison on one B200.
    python tools/ljsde_bench.py [--rows 128] [--window 32] [--iterations 200]
    python tools/ljsde_bench.py --rows 1200 --period 32 --seed 501 --no-reference
        (acceptance.cpp:301-323, criterion 5's 1200^2 leg: an hour for the reference's
        single-thread protocol, so only the device pair runs)"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2205_02646_b200 as tq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=128)
ap.add_argument("--window", type=int, default=32)
ap.add_argument("--iterations", type=int, default=200)
ap.add_argument("--period", type=int, default=8)
ap.add_argument("--seed", type=int, default=301)
ap.add_argument("--no-reference", action="store_true")
a = ap.parse_args()
gt = tq.synthetic_image(a.rows, a.rows, a.seed)
pat = tq.generate_pattern(7, a.period)
frame = tq.simulate_measurement(gt, pat)
ref = oracle.Reference()
res = {"image": [a.rows, a.rows], "window": a.window, "iterations": a.iterations,
       "period": a.period, "seed": a.seed, "host_cores": ref.hardware_threads()}
want_l = None
for algo in (() if a.no_reference else ("ljsde", "rljsde")):
    t = time.perf_counter()
    want, sec = ref.reconstruct_algo(frame, pat.opaque, a.period, algo, window=a.window,
                                     iterations=a.iterations, threads=0)
    res[f"reference_{algo}_s"] = sec
    res[f"reference_{algo}_wall_s"] = time.perf_counter() - t
    if algo == "ljsde":
        want_l = want
cfgL = tq.ReconstructionConfig(window=a.window, max_iterations=a.iterations, clip_output=False,
                               algorithm=tq.ALGO_LJSDE)
with tq.Plan(pat, cfgL) as plan:
    plan.reconstruct(frame)
    r = plan.reconstruct(frame)
res["gpu_ljsde_s"] = r.seconds
if want_l is not None:
    res["gpu_ljsde_max_abs_vs_reference"] = float(np.abs(r.output - want_l).max())
for name, comp in (("gpu_rljsde_fp64_s", tq.COMPUTE_FP64), ("gpu_rljsde_fp32_s", tq.COMPUTE_FP32)):
    cfg = tq.ReconstructionConfig(window=a.window, max_iterations=a.iterations, clip_output=False,
                                  compute=comp)
    with tq.Plan(pat, cfg) as plan:
        plan.reconstruct(frame)
        rr = plan.reconstruct(frame)
    res[name] = rr.seconds
    if comp == tq.COMPUTE_FP64:
        res["gpu_l_vs_rl_fp64_max_abs"] = float(np.abs(rr.output - r.output).max())
if want_l is not None:
    res["gpu_ljsde_speedup_vs_reference_ljsde"] = res["reference_ljsde_s"] / res["gpu_ljsde_s"]
res["gpu_rl_fp64_speedup_vs_gpu_ljsde"] = res["gpu_ljsde_s"] / res["gpu_rljsde_fp64_s"]
res["gpu_rl_fp32_speedup_vs_gpu_ljsde"] = res["gpu_ljsde_s"] / res["gpu_rljsde_fp32_s"]
print(json.dumps(res))
