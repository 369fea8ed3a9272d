#!/usr/bin/env bash
# Round-2 closing evidence (under gpurun): everything in r02_final.sh plus the parity
# table of the final build and one `ncu --set full` capture of the product kernel.
set -u
tag=${1:-r02z}
bash tools/r02_final.sh $tag
python tools/parity_r02.py --out gpurun_out/${tag}_parity.jsonl > gpurun_out/${tag}_parity.log 2>&1
cmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve_f32 -c 1 \
    -o /tmp/${tag}_solve $cmd > gpurun_out/${tag}_ncu_full.log 2>&1
if [ -f /tmp/${tag}_solve.ncu-rep ]; then
  cp /tmp/${tag}_solve.ncu-rep gpurun_out/
  ncu -i /tmp/${tag}_solve.ncu-rep --page raw --csv > gpurun_out/${tag}_solve_raw.csv
fi
ls gpurun_out | grep $tag | wc -l
