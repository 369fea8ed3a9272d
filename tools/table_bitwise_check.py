import sys, numpy as np
sys.path.insert(0,'.')
import oracle, paper_2205_02646_b200 as tq
ref=oracle.Reference()
for (W,P,seed,o) in [(8,8,5,(3,5)),(16,32,7,(6,10)),(32,8,7,(14,14)),(20,4,9,(0,2))]:
    pat=tq.generate_pattern(seed,P,2)
    with tq.Plan(pat, tq.ReconstructionConfig(window=W, block=2, compute=tq.COMPUTE_FP64)) as plan:
        got=plan.export_tables(*o)
    want=ref.precompute(pat.opaque,P,o[0],o[1],W)
    print(W,P, "b eq", np.array_equal(got["b"],want["b"]), "c eq", np.array_equal(got["c"],want["c"]), "d eq", np.array_equal(got["d"],want["d"]), "c maxdiff", np.abs(got["c"]-want["c"]).max())
