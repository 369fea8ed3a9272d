import sys, numpy as np
sys.path.insert(0,'.')
import oracle, paper_2205_02646_b200 as tq
ref=oracle.Reference()
for (W,P,B,o) in [(8,4,2,(0,7)),(8,4,2,(0,9)),(8,4,2,(0,28)),(20,4,4,(0,4))]:
    pat=tq.generate_pattern(11,P,B)
    with tq.Plan(pat, tq.ReconstructionConfig(window=W, block=B, compute=tq.COMPUTE_FP64)) as plan:
        got=plan.export_tables(*o)
    want=ref.precompute(pat.opaque,P,o[0],o[1],W)
    print(W,P,o, "L", got["L"], want["L"], "b", np.array_equal(got["b"],want["b"]), "c", np.array_equal(got["c"],want["c"]), "d", np.array_equal(got["d"],want["d"]), np.abs(got["c"]-want["c"]).max(), np.abs(got["b"]-want["b"]).max())
