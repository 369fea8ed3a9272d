"""Turn the CSV exports of tools/profile_round.sh (gpurun_out/<tag>_*) into the tracked
evidence under profiles/: the launch list with per-kernel shares, the ncu --set full
summary of the solve kernel (SOL, stalls, instruction mix per warp-iteration, top
stall sites) and ncu_traffic.json (DRAM bytes per launch, read by bench.py).

    python tools/make_profiles.py r01b [--out r01] [--blocks 518400 --iters 200]
"""
import argparse
import collections
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def launches(tag, out):
    text = [ln for ln in open(os.path.join(G, f"{tag}_launches.csv")) if not ln.startswith("==")]
    rows = list(csv.reader(text))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]]
        ns = float(r[ix["Metric Value"]])
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values())
    lines = ["# ncu launch list of `python bench.py --steps 2 --warmup 1 --no-cpu-baseline` "
             "(4K, P=8, 1 B200)",
             "# gpu__time_duration.sum (ns), --clock-control none; cold-cache serialised launches: "
             "compare SHARES",
             f"{'kernel':<72} {'launches':>8} {'total_us':>12} {'mean_us':>10} {'share':>7}"]
    for name, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:72]:<72} {n:>8} {ns / 1e3:>12.1f} {ns / n / 1e3:>10.1f} "
                     f"{100 * ns / tot:>6.2f}%")
    open(os.path.join(P, f"{out}_launches_bench_4k.txt"), "w").write("\n".join(lines) + "\n")
    return agg


def full(tag, out, witers):
    det = list(csv.reader(open(os.path.join(G, f"{tag}_solve_details.csv"))))
    hdr = det[0]
    keep = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput",
            "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
            "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
            "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler",
            "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Executed Instructions", "Dynamic Shared Memory Per Block"]
    lines, seen = [], set()
    kname = None
    for row in det[1:]:
        d = dict(zip(hdr, row))
        kname = d.get("Kernel Name", kname)
        m = d.get("Metric Name")
        if m in keep and m not in seen:
            seen.add(m)
            lines.append(f"{m:<40} {d['Metric Value']:>16} {d.get('Metric Unit', '')}")
    raw = list(csv.reader(open(os.path.join(G, f"{tag}_solve_raw.csv"))))
    rh, ru, rv = raw[0], raw[1], raw[2]
    rawd = {}
    for name in ["dram__bytes_read.sum", "dram__bytes_write.sum",
                 "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                 "l1tex__throughput.avg.pct_of_peak_sustained_active",
                 "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
                 "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]:
        if name in rh:
            i = rh.index(name)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ru[i], 1)
            rawd[name] = float(rv[i]) * scale
            lines.append(f"{name:<64} {rv[i]:>18} {ru[i]}")
    # instruction mix + stall mix from the source page
    src = list(csv.reader(open(os.path.join(G, f"{tag}_solve_src.csv"))))
    sh, sd = src[1], src[2:]
    ix = {h: i for i, h in enumerate(sh)}
    stalls = [h for h in sh if h.startswith("stall_") and "Not Issued" not in h]
    mix, st = collections.Counter(), collections.Counter()
    tot = 0
    sites = []
    for r in sd:
        ex = int(r[ix["Instructions Executed"]] or 0)
        op = r[1].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        mix[o.split(".")[0]] += ex
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        tot += s
        for h in stalls:
            st[h[6:]] += int(r[ix[h]] or 0)
        sites.append((s, r[1].strip()[:60],
                      max(stalls, key=lambda h: int(r[ix[h]] or 0))[6:]))
    lines.append("stall mix: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in st.most_common(8)))
    lines.append(f"instructions per warp-iteration: {sum(mix.values()) / witers:.1f}")
    lines.append("  " + ", ".join(f"{o} {c / witers:.1f}" for o, c in mix.most_common(18)))
    lines.append("top stall sites (share of samples, instruction, dominant reason):")
    for s, ins, why in sorted(sites, reverse=True)[:12]:
        lines.append(f"  {100 * s / tot:5.2f}%  {ins:<60} {why}")
    header = [f"# ncu --set full --clock-control none, one launch of {kname}",
              "# command: python bench.py --steps 2 --warmup 1 --no-cpu-baseline (4K frame, P=8)"]
    open(os.path.join(P, f"{out}_ncu_solve_4k.txt"), "w").write("\n".join(header + lines) + "\n")
    rd, wr = int(rawd["dram__bytes_read.sum"]), int(rawd["dram__bytes_write.sum"])
    json.dump({"workload": "4k", "blocks": 518400, "kernel": kname,
               "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
               "source": f"profiles/{out}_ncu_solve_4k.txt (ncu --set full, bench.py --steps 2 "
                         f"--warmup 1)"},
              open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)


def raw_lines(tag, out):
    """The bench lines of tools/evidence.sh (headline, reference arm, period sweep, video,
    L-JSDE comparison) copied under profiles/ and the sweep/video summary refreshed."""
    import re
    import shutil

    def cp(src, dst, last_line=False):
        path = os.path.join(G, src)
        if not os.path.exists(path):
            return None
        text = open(path).read().strip().splitlines()[-1] if last_line else None
        if last_line:
            open(os.path.join(P, dst), "w").write(text + "\n")
        else:
            shutil.copy(path, os.path.join(P, dst))
        return json.loads(open(os.path.join(P, dst)).read().strip().splitlines()[-1])

    cp(f"{tag}_bench.json", f"{out}_bench_4k.json", True)
    cp(f"{tag}_bench_reference.json", f"{out}_bench_reference_4k.json", True)
    sweep = {p: cp(f"{tag}_sweep_p{p}.json", f"{out}_bench_1mp_p{p}.json", True) for p in (4, 8, 16, 32)}
    v = cp(f"{tag}_video.json", f"{out}_bench_video.json", True)
    lj = cp(f"{tag}_ljsde.json", f"{out}_ljsde_vs_rljsde.json", True)
    doc_path = os.path.join(P, f"{out}_period_sweep_video.md")
    if not os.path.exists(doc_path) or any(x is None for x in sweep.values()) or v is None or lj is None:
        return
    doc = open(doc_path).read()
    doc = re.sub(r"Files: `gpurun_out/\w+_\*` of `bash tools/evidence.sh \w+`[^)]*\)",
                 f"Files: `gpurun_out/{tag}_*` of `bash tools/evidence.sh {tag}` (copied here as this summary)", doc)
    names = {4: "2x2 (P=4)", 8: "4x4 (P=8)", 16: "8x8 (P=16)", 32: "16x16 (P=32)"}
    for p, d in sweep.items():
        c = d["cpu_baseline"]
        row = (f"| {names[p]} | {d['value']:.1f} | {d['e2e']['value']:.1f} | {d['warm_seconds']:.2f} | "
               f"{c['value']:.3f} ({c['cores']} cores) | {d['e2e']['value'] / c['value']:.0f}x | "
               f"{d['roofline']['frac']:.3f} / {d['roofline']['frac_nominal']:.3f} |")
        doc = re.sub(r"^\| " + re.escape(names[p]) + r" \|.*$", row, doc, flags=re.M)
    doc = re.sub(r"\| device-resident frames \(`value`\) \| [0-9.]+ \| [0-9.]+ \|",
                 f"| device-resident frames (`value`) | {v['value']:.1f} | {v['ms_per_step']:.1f} |", doc)
    doc = re.sub(r"(\| host frames through `tqsb_reconstruct_batch`[^|]*\|) [0-9.]+ \| [0-9.]+ \|",
                 lambda m: f"{m.group(1)} {v['e2e']['value']:.1f} | {v['e2e']['ms_per_step']:.1f} |", doc)
    doc = re.sub(r"(\| sensor in the loop[^|]*\|) [0-9.]+ \| [0-9.]+ \|",
                 lambda m: f"{m.group(1)} {v['device_stream']['value']:.1f} | {v['device_stream']['ms_per_step']:.1f} |", doc)
    doc = re.sub(r"Roofline frac [0-9.]+ of the measured FFMA2 peak.",
                 f"Roofline frac {v['roofline']['frac']:.3f} of the measured FFMA2 peak.", doc)
    doc = re.sub(r"\| reference L-JSDE \| [0-9.]+ \|", f"| reference L-JSDE | {lj['reference_ljsde_s']:.3f} |", doc)
    doc = re.sub(r"\| reference RL-JSDE \(block phase\) \| [0-9.]+ \|",
                 f"| reference RL-JSDE (block phase) | {lj['reference_rljsde_s']:.4f} |", doc)
    doc = re.sub(r"\| device L-JSDE \(fp64, reference summation order\) \| [0-9.]+ \| [0-9.]+x faster; max-abs [0-9.e-]+",
                 f"| device L-JSDE (fp64, reference summation order) | {lj['gpu_ljsde_s']:.3f} | "
                 f"{lj['gpu_ljsde_speedup_vs_reference_ljsde']:.1f}x faster; max-abs {lj['gpu_ljsde_max_abs_vs_reference']:.1e}", doc)
    doc = re.sub(r"\| device RL-JSDE fp64 parity mode \| [0-9.]+ \| L <-> RL max-abs [0-9.e-]+",
                 f"| device RL-JSDE fp64 parity mode | {lj['gpu_rljsde_fp64_s']:.4f} | L <-> RL max-abs {lj['gpu_l_vs_rl_fp64_max_abs']:.1e}", doc)
    doc = re.sub(r"\| device RL-JSDE fp32 product path \| [0-9.]+ \| [0-9]+x faster",
                 f"| device RL-JSDE fp32 product path | {lj['gpu_rljsde_fp32_s']:.5f} | {lj['gpu_rl_fp32_speedup_vs_gpu_ljsde']:.0f}x faster", doc)
    open(doc_path, "w").write(doc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--out", default="r01")
    ap.add_argument("--blocks", type=int, default=518400)
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    launches(a.tag, a.out)
    full(a.tag, a.out, a.blocks * a.iters)
    raw_lines(a.tag, a.out)


if __name__ == "__main__":
    main()
