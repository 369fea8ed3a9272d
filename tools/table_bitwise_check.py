"""Device-built fp64 tables (K1, tables.cu) against the reference's precompute_kernels:
bitwise equality of B, C, D for a set of classes (odd and even origins, several W / P).
    python tools/table_bitwise_check.py"""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle  # noqa: E402
import paper_2205_02646_b200 as tq  # noqa: E402

ref = oracle.Reference()
for W, P, B, seed, o in [(8, 8, 2, 5, (3, 5)), (16, 32, 2, 7, (6, 10)), (32, 8, 2, 7, (14, 14)),
                         (20, 4, 2, 9, (0, 2)), (8, 4, 2, 11, (0, 7)), (8, 4, 2, 11, (1, 5)),
                         (20, 4, 4, 11, (0, 4))]:
    pat = tq.generate_pattern(seed, P, B)
    with tq.Plan(pat, tq.ReconstructionConfig(window=W, block=B, compute=tq.COMPUTE_FP64)) as plan:
        got = plan.export_tables(*o)
    want = ref.precompute(pat.opaque, P, o[0], o[1], W)
    print(f"W={W} P={P} origin={o} L={got['L']}/{want['L']}",
          "B", np.array_equal(got["b"], want["b"]), "C", np.array_equal(got["c"], want["c"]),
          "D", np.array_equal(got["d"], want["d"]))
