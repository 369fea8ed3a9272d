#!/usr/bin/env bash
# Round evidence on one B200 (run under gpurun): the bench line, the ncu launch list
# of the same bench command, and one `ncu --set full` capture of the solve kernel,
# exported as CSV into gpurun_out/ (tools/make_profiles.py turns them into profiles/).
set -u
tag=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
cmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$cmd > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv $cmd > gpurun_out/${tag}_ncu_list.log 2>&1
$cmd > gpurun_out/${tag}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_solve_f32 -c 1 \
    -o /tmp/${tag}_solve $cmd > gpurun_out/${tag}_ncu_full.log 2>&1
if [ -f /tmp/${tag}_solve.ncu-rep ]; then
  ncu -i /tmp/${tag}_solve.ncu-rep --page details --csv > gpurun_out/${tag}_solve_details.csv
  ncu -i /tmp/${tag}_solve.ncu-rep --page raw --csv > gpurun_out/${tag}_solve_raw.csv
  ncu -i /tmp/${tag}_solve.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_solve_src.csv
fi
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>&1
ls -la gpurun_out
