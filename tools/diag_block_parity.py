"""Locate blocks where the device fp64 mode and the reference disagree and compare
their greedy paths (device block trace vs the reference's rljsde_block hook).
    python tools/diag_block_parity.py W B P rows [iterations]"""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle  # noqa: E402
import paper_2205_02646_b200 as tq  # noqa: E402

W, B, P, rows = (int(x) for x in sys.argv[1:5])
it = int(sys.argv[5]) if len(sys.argv) > 5 else 60
ref, orc = oracle.Reference(), oracle.Oracle()
img = tq.synthetic_image(rows, rows + 2 * B, 500 + W + B)
pat = tq.generate_pattern(11, P, B)
frame = tq.simulate_measurement(img, pat)
want, _ = ref.reconstruct(frame, pat.opaque, P, window=W, block=B, iterations=it, clip=False)
cfg = tq.ReconstructionConfig(window=W, block=B, max_iterations=it, clip_output=False,
                              compute=tq.COMPUTE_FP64)
M, N = want.shape
lead = (W - B) // 2
with tq.Plan(pat, cfg) as plan:
    got = plan.reconstruct(frame).output
    d = np.abs(got - want)
    bad = []
    for br in range(0, M, B):
        for bc in range(0, N, B):
            e = d[br:br + B, bc:bc + B].max()
            if e > 1e-9:
                orow = min(max(br - lead, 0), M - W)
                ocol = min(max(bc - lead, 0), N - W)
                bad.append((br, bc, orow, ocol, e))
    print(f"{len(bad)} of {(M // B) * (N // B)} blocks differ; max {d.max():.3g}")
    for b in bad[:8]:
        print("  block", b[:2], "origin", b[2:4], "class", (b[2] % P, b[3] % P), f"err {b[4]:.3g}")
    if bad:
        br, bc, orow, ocol, _ = bad[0]
        y = orc.gather(frame, orow, ocol, W)
        dp, dg, dwin = plan.block_trace(orow, ocol, y)
        rp, rg, rwin = ref.block_trace(pat.opaque, P, orow, ocol, W, y, iterations=it)
        n = min(len(dp), len(rp))
        first = next((i for i in range(n) if dp[i] != rp[i]), None)
        print("  picks: device", len(dp), "reference", len(rp), "first fork", first)
        if first is not None:
            print("   device   ", dp[max(0, first - 2):first + 3], dg[first])
            print("   reference", rp[max(0, first - 2):first + 3], rg[first])
        pre = first if first is not None else n
        print("  gd bitwise equal before the fork:", bool(np.array_equal(dg[:pre], rg[:pre])),
              "max diff", np.abs(dg[:pre] - rg[:pre]).max() if pre else 0.0)
        neq = [i for i in range(pre) if dg[i] != rg[i]]
        print("  first gd difference at iteration", neq[0] if neq else None,
              (dg[neq[0]], rg[neq[0]]) if neq else "")
        # q: the device's frequency weights vs the reference's
        qd = plan.frequency_weights() if hasattr(plan, "frequency_weights") else None
        qr = ref.frequency_weights(W)
        qo = orc.frequency_weights(W)
        print("  q oracle == reference:", bool(np.array_equal(qo, qr)))
        k0 = first
        if k0 is not None:
            # the two candidates' scores on the reference path, from the oracle's tables
            # and a restatement of the recursion (exact reference arithmetic via numpy fma-free
            # is not bitwise, so only the relative gap is printed)
            pass
        print("  gd max diff (common prefix)", np.abs(dg[:n] - rg[:n]).max() if n else None,
              " window max diff", np.abs(dwin - rwin).max())
