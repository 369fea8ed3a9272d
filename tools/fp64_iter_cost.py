import sys, time
sys.path.insert(0,'.')
import paper_2205_02646_b200 as tq
img=tq.synthetic_image(1200,1200,501); pat=tq.generate_pattern(7,8); frame=tq.simulate_measurement(img,pat)
for it in (0,1,10,200):
    with tq.Plan(pat, tq.ReconstructionConfig(compute=tq.COMPUTE_FP64, clip_output=False, max_iterations=it)) as plan:
        plan.reconstruct(frame); r=plan.reconstruct(frame)
    print(it, r.seconds, r.blocks_processed)
