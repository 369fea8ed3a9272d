"""Where the pageable drop-in call spends its time beyond the pinned one (4K frame):
pinned/pageable input x pinned/fresh-pageable/reused-pageable output, through
Plan.reconstruct (tqsb_reconstruct_with). Prints one JSON line per combination."""
import ctypes
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_02646_b200 as tq  # noqa: E402


def pinned(shape):
    n = int(np.prod(shape))
    p = tq.lib.tqsb_host_alloc(8 * n)
    return np.ctypeslib.as_array((ctypes.c_double * n).from_address(p)).reshape(shape)


def main():
    gt = tq.synthetic_image(2160, 3840, 501)
    pat = tq.generate_pattern(7, 8)
    frame = tq.simulate_measurement(gt, pat)
    plan = tq.Plan(pat, tq.ReconstructionConfig())
    fin_pin = pinned(frame.shape)
    fin_pin[...] = frame
    out_pin = pinned(gt.shape)
    out_reuse = np.empty(gt.shape)
    for name, fin, outf in [("pinned_in/pinned_out", fin_pin, lambda: out_pin),
                            ("pageable_in/pinned_out", frame, lambda: out_pin),
                            ("pinned_in/fresh_pageable_out", fin_pin, lambda: None),
                            ("pinned_in/reused_pageable_out", fin_pin, lambda: out_reuse),
                            ("pageable_in/fresh_pageable_out", frame, lambda: None)]:
        ts, dev = [], []
        for i in range(8):
            t = time.perf_counter()
            r = plan.reconstruct(fin, out=outf())
            if i >= 2:
                ts.append(time.perf_counter() - t)
                dev.append(r.seconds)
        print(json.dumps({"case": name, "ms": round(statistics.mean(ts) * 1e3, 3),
                          "device_ms": round(statistics.mean(dev) * 1e3, 3),
                          "min_ms": round(min(ts) * 1e3, 3)}), flush=True)


if __name__ == "__main__":
    main()
