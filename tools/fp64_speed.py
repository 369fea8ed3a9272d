"""Block-phase time of the fp64 parity mode on one image (second plan call).
    python tools/fp64_speed.py [rows] [period]"""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2205_02646_b200 as tq  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
P = int(sys.argv[2]) if len(sys.argv) > 2 else 32
img = tq.synthetic_image(rows, rows, 501)
pat = tq.generate_pattern(7, P)
frame = tq.simulate_measurement(img, pat)
with tq.Plan(pat, tq.ReconstructionConfig(compute=tq.COMPUTE_FP64, clip_output=False)) as plan:
    plan.reconstruct(frame)
    r = plan.reconstruct(frame)
print(f"fp64 mode {rows}x{rows} P={P}: {r.seconds:.4f} s = {rows * rows / 1e6 / r.seconds:.2f} MP/s")
import time  # noqa: E402
t = time.perf_counter()
with tq.Plan(pat, tq.ReconstructionConfig(compute=tq.COMPUTE_FP64, clip_output=False)) as plan:
    plan.reconstruct(frame)
    t1 = time.perf_counter()
    r = plan.reconstruct(frame)
    t2 = time.perf_counter()
print(f"  wall: first call {t1 - t:.2f} s, second call {t2 - t1:.3f} s (report.seconds {r.seconds:.3f}, "
      f"blocks {r.blocks_processed})")
