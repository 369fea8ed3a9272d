"""Kernel-variant A/B driver: time k_solve_f32 of several libtqsb builds on the same
device-resident frame and compare each output with the first library's and with
the fp64 device path (parity proxy: max |d| and PSNR delta vs ground truth).

    python tools/variants.py --libs libtqsb.so libtqsb_keys.so [--rows 2160 --cols 3840]

Each library runs in its own subprocess (TQSB_LIB selects it).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2205_02646_b200")


def child(a):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import paper_2205_02646_b200 as tq
    gt = tq.synthetic_image(a.rows, a.cols, a.seed)
    pat = tq.generate_pattern(7, a.period)
    frame = tq.simulate_measurement(gt, pat)
    plan = tq.Plan(pat, tq.ReconstructionConfig(clip_output=False,
                                                hot_columns=int(os.environ.get("TQSB_HOT", "-1"))))
    plan.warm(*frame.shape)
    d_frame = torch.from_numpy(frame).cuda()
    d_out = torch.empty((a.rows, a.cols), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ms = []
    for i in range(a.reps + 1):
        flush.fill_(i & 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        plan.reconstruct_device(d_frame.data_ptr(), frame.shape[0], frame.shape[1],
                                d_out.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        if i:
            ms.append(e0.elapsed_time(e1))
    out = d_out.cpu().numpy()
    np.save(a.save, out)
    psnr = 10 * np.log10(1.0 / np.mean((out - gt) ** 2))
    print(json.dumps({"lib": os.environ.get("TQSB_LIB"), "ms": ms, "min_ms": min(ms),
                      "psnr": psnr}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="+", default=["libtqsb.so"])
    ap.add_argument("--rows", type=int, default=2160)
    ap.add_argument("--cols", type=int, default=3840)
    ap.add_argument("--seed", type=int, default=501)
    ap.add_argument("--period", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--save", default="")
    a = ap.parse_args()
    if a.child:
        return child(a)
    import numpy as np
    res = []
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for i, lib in enumerate(a.libs):
        save = f"/tmp/variant_{i}.npy"
        env = dict(os.environ, TQSB_LIB=os.path.join(PKG, lib))
        cmd = [sys.executable, __file__, "--child", "--rows", str(a.rows), "--cols", str(a.cols),
               "--seed", str(a.seed), "--period", str(a.period), "--reps", str(a.reps),
               "--save", save]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True)
        if r.returncode != 0:
            print(lib, "FAILED", r.stderr[-2000:])
            continue
        j = json.loads(r.stdout.strip().splitlines()[-1])
        out = np.load(save)
        if res:
            base = np.load("/tmp/variant_0.npy")
            d = np.abs(out - base)
            j["max_abs_vs_first"] = float(d.max())
            j["px_gt_1e-4_vs_first"] = int((d > 1e-4).sum())
            j["dpsnr_vs_first"] = j["psnr"] - res[0]["psnr"]
        res.append(j)
        print(json.dumps(j), flush=True)


if __name__ == "__main__":
    main()
