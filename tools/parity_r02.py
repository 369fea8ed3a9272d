"""Parity table of the fp32 product path against the unmodified reference
(oracle/_ref, fp64 default, clip off) at every BASELINE.json config at its stated
size, plus the 1 MP U[0,1) stress input and a non-block-multiple frame.
For each input the reference's own Precision::Single run is measured against its
Double run too, so the fp32 deviation is set beside the reference's own.

    python tools/parity_r02.py [--out gpurun_out/parity_r02.jsonl] [--quick]

Prints / writes one JSON line per case: max_abs, dpsnr (dB), px_gt_1e4 for
ours-vs-double and single-vs-double. Test infrastructure (imports oracle/).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2205_02646_b200 as tq  # noqa: E402


def psnr(gt, x):
    return float(10 * np.log10(1.0 / np.mean((gt - x) ** 2)))


def cmp(x, want, gt):
    d = np.abs(x - want)
    return dict(max_abs=float(d.max()), dpsnr=psnr(gt, x) - psnr(gt, want),
                px_gt_1e4=int((d > 1e-4).sum()), px=int(d.size))


def cases(quick):
    yield "c0_128_p8", [(tq.synthetic_image(128, 128, 301), 8)]
    yield "c1_1mp_p8", [(tq.synthetic_image(1024, 1024, 401), 8)]
    if not quick:
        yield "c2_4k_p8", [(tq.synthetic_image(2160, 3840, 501), 8)]
    for P in (4, 16, 32):
        yield f"c3_1mp_p{P}", [(tq.synthetic_image(1024, 1024, 401), P)]
    yield "c4_video_1mp_p16_x4", [(tq.synthetic_image(1024, 1024, 1000 + i), 16) for i in range(4)]
    yield "noise_1mp_p8", [(np.random.default_rng(401).random((1024, 1024)), 8)]
    yield "noise_128_p8", [(np.random.default_rng(5).random((128, 128)), 8)]
    yield "odd_1082x1922_p8", [(tq.synthetic_image(1082, 1922, 403), 8)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_r02.jsonl"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--no-single", action="store_true")
    args = ap.parse_args()
    ref = oracle.Reference()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fo:
        for name, items in cases(args.quick):
            P = items[0][1]
            pat = tq.generate_pattern(7, P)
            frames = [tq.simulate_measurement(gt, pat) for gt, _ in items]
            t0 = time.time()
            wants = [ref.reconstruct(f, pat.opaque, P, clip=False, threads=0)[0] for f in frames]
            t_ref = time.time() - t0
            singles = None if args.no_single else [
                ref.reconstruct(f, pat.opaque, P, clip=False, threads=0, double=False)[0]
                for f in frames]
            cfg = tq.ReconstructionConfig(clip_output=False)
            with tq.Plan(pat, cfg) as plan:
                if len(frames) > 1:
                    outs = plan.reconstruct_batch(frames).output
                else:
                    outs = [plan.reconstruct(frames[0]).output]
            gts = [gt for gt, _ in items]
            allo, allw, allg = (np.concatenate([a.ravel() for a in v]) for v in (outs, wants, gts))
            row = dict(case=name, period=P, frames=len(frames), shape=list(items[0][0].shape),
                       ref_seconds=round(t_ref, 2), fp32_vs_ref=cmp(allo, allw, allg))
            if singles is not None:
                alls = np.concatenate([a.ravel() for a in singles])
                row["ref_single_vs_ref"] = cmp(alls, allw, allg)
            row["per_frame_max_abs"] = [float(np.abs(o - w).max()) for o, w in zip(outs, wants)]
            print(json.dumps(row), flush=True)
            fo.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
