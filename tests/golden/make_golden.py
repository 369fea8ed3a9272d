"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
library (oracle/_ref, compiled from /root/reference/proj by oracle/build_ref.sh).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are committed; the GPU box never needs /root/reference.
Every case names the reference call it pins.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    ref = oracle.Reference()
    fx = {}
    # generate_pattern (grid.cpp:8-26)
    for seed, P in [(7, 4), (7, 8), (7, 16), (7, 32), (11, 32), (13, 32), (5, 8)]:
        fx[f"pattern_s{seed}_p{P}"] = ref.generate_pattern(seed, P, 2 if P % 4 else 4)
    # synthetic_image (tests/support/synthetic.cpp:9-80), simulate (grid.cpp:46-66)
    img = ref.synthetic_image(64, 64, 8)
    fx["synthetic_64_s8"] = img
    pat32 = ref.generate_pattern(7, 32)
    frame = ref.simulate(img, pat32, 32)
    fx["frame_64_s8_p32"] = frame
    # reconstruct (pipeline.cpp:62-185): test_pipeline.cpp:219-236 configuration
    out, rep = ref.reconstruct(frame, pat32, 32, window=16, block=4, iterations=100,
                               clip=False, threads=1)
    fx["recon_64_s8_p32_w16_it100"] = out
    fx["recon_64_s8_p32_w16_it100_census"] = np.array(
        [rep.blocks, rep.classes_total, rep.classes_interior, rep.cache_hits, rep.cache_misses])
    # the BASELINE oracle config: 128x128, period 4x4 cells (P = 8), reference defaults
    img128 = ref.synthetic_image(128, 128, 301)
    pat8 = ref.generate_pattern(7, 8)
    frame128 = ref.simulate(img128, pat8, 8)
    out128, rep128 = ref.reconstruct(frame128, pat8, 8, clip=False, threads=0,
                                     reference=img128)
    fx["frame_128_s301_p8"] = frame128
    fx["recon_128_s301_p8_default_noclip"] = out128
    fx["recon_128_s301_p8_default_noclip_psnr"] = np.array([rep128.psnr_db])
    # tables of one toy class (precompute_kernels, rljsde.cpp:186-201), W = 8, odd origin
    pat_toy = ref.generate_pattern(5, 8, 2)
    t = ref.precompute(pat_toy, 8, 3, 5, 8)
    fx["tables_w8_p8_s5_o3_5_b"] = t["b"]
    fx["tables_w8_p8_s5_o3_5_c"] = t["c"]
    fx["tables_w8_p8_s5_o3_5_d"] = t["d"]
    # one production block's greedy path (rljsde_block + IterationHook)
    y = np.array([frame128[r, c] for r in range(7, 23) for c in range(7, 23)])
    picks, gd, win = ref.block_trace(pat8, 8, 14, 14, 32, y)
    fx["trace_128_s301_p8_o14_14_picks"] = picks
    fx["trace_128_s301_p8_o14_14_gd"] = gd
    fx["trace_128_s301_p8_o14_14_window"] = win
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **fx)
    print("wrote", os.path.join(OUT, "golden.npz"), len(fx), "arrays")


if __name__ == "__main__":
    main()
