"""One line per library from tools/variants.py output: min ms, max-abs vs the first library, PSNR.

    python tools/variants.py --libs a.so b.so | python tools/variants_summary.py
"""
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300].rstrip()); continue
    print(d["lib"].split("/")[-1], round(d.get("min_ms",0),3), "maxabs_vs_first", d.get("max_abs_vs_first"), "psnr", d.get("psnr"))
