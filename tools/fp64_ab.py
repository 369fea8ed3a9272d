"""A/B of fp64-mode (k_solve_f64r) library variants in one process each, same box:
block-phase seconds at nu = 0 (init + placement) and nu = 200.
    python tools/fp64_ab.py libtqsb.so libtqsb_x.so ... [--rows 1200 --period 8]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(rows, period):
    sys.path.insert(0, ROOT)
    import paper_2205_02646_b200 as tq
    img = tq.synthetic_image(rows, rows, 501)
    pat = tq.generate_pattern(7, period)
    frame = tq.simulate_measurement(img, pat)
    res = {}
    for nu in (0, 200):
        cfg = tq.ReconstructionConfig(compute=tq.COMPUTE_FP64, clip_output=False, max_iterations=nu)
        with tq.Plan(pat, cfg) as plan:
            plan.reconstruct(frame)
            ts = [plan.reconstruct(frame).seconds for _ in range(3)]
        res[f"nu{nu}_s"] = min(ts)
    res["mps"] = rows * rows / 1e6 / res["nu200_s"]
    print(json.dumps(res))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--rows", type=int, default=1200)
    ap.add_argument("--period", type=int, default=8)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.rows, a.period)
        sys.exit(0)
    for rep in range(2):
        for lib in a.libs:
            env = dict(os.environ, TQSB_LIB=os.path.join(ROOT, "paper_2205_02646_b200", lib))
            out = subprocess.run([sys.executable, __file__, "--child", "--rows", str(a.rows), "--period",
                                  str(a.period)], env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(json.dumps({"lib": lib, "rep": rep, "rows": a.rows, "period": a.period,
                              **(json.loads(line) if line.startswith("{") else {"err": line})}), flush=True)
