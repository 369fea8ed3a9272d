"""Summarise tools/ncu3.sh CSV exports: key raw metrics, instruction mix per
warp-iteration, and stall samples per code region of the hot loop.
    python tools/ncu_view.py VARIANT [--iters N] [--dump]"""
import collections
import csv
import sys

v = sys.argv[1]
iters = 65536 * 200
rows = list(csv.reader(open(f"gpurun_out/raw_{v}.csv")))
raw = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
          "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread"]:
    print(f"{k:66s} {raw.get(k)}")
rows = list(csv.reader(open(f"gpurun_out/src_{v}.csv")))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
mix = collections.Counter()
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
st = collections.Counter()
tot = 0
for r in data:
    ex = int(r[ix["Instructions Executed"]] or 0)
    op = r[1].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    mix[o.split(".")[0]] += ex
    for h in stalls:
        st[h[6:]] += int(r[ix[h]] or 0)
    tot += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
print("instr / warp-iteration:", round(sum(mix.values()) / iters, 1))
print("  ", ", ".join(f"{o} {c / iters:.1f}" for o, c in mix.most_common(22)))
print("stalls:", ", ".join(f"{k} {100 * c / tot:.1f}%" for k, c in st.most_common(10)))
if "--dump" in sys.argv:
    mx = max(int(r[ix["Instructions Executed"]] or 0) for r in data)
    for n, r in enumerate(data):
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ex = int(r[ix["Instructions Executed"]] or 0)
        if ex > 0.3 * mx or s > tot * 0.004:
            top = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
            print(f"{n:5d} {s:6d} {ex:9d} {r[1].strip()[:58]:58s} {top[0][1]}:{top[0][0]} {top[1][1]}:{top[1][0]}")
