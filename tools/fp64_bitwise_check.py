"""How close is the fp64 parity mode to the reference? Max-abs and bitwise-equal pixel
share over a grid of configurations (W, B, P, image), clip off, nu = 60.
    python tools/fp64_bitwise_check.py"""
import json
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle  # noqa: E402
import paper_2205_02646_b200 as tq  # noqa: E402

ref = oracle.Reference()
rows_out = []
for W, B, P, rows in [(8, 2, 4, 32), (12, 4, 8, 48), (20, 4, 4, 64), (18, 6, 12, 72), (24, 8, 8, 64),
                      (30, 2, 4, 64), (32, 8, 8, 64), (16, 16, 16, 48), (32, 4, 8, 128), (32, 4, 32, 128),
                      (16, 4, 16, 96), (36, 4, 4, 72)]:
    img = tq.synthetic_image(rows, rows + 2 * B, 500 + W + B)
    pat = tq.generate_pattern(11, P, B)
    frame = tq.simulate_measurement(img, pat)
    want, _ = ref.reconstruct(frame, pat.opaque, P, window=W, block=B, iterations=60, clip=False,
                              threads=0)
    got = tq.reconstruct(frame, pat, tq.ReconstructionConfig(
        window=W, block=B, max_iterations=60, clip_output=False, compute=tq.COMPUTE_FP64)).output
    d = np.abs(got - want)
    r = dict(W=W, B=B, P=P, rows=rows, max_abs=float(d.max()), bitwise_px=float((d == 0).mean()))
    rows_out.append(r)
    print(json.dumps(r), flush=True)
