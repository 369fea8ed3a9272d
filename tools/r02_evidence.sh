#!/usr/bin/env bash
# Round-2 evidence on one B200 (run under gpurun): bench line (N=1), a 2-rank torchrun
# on the same GPU (gloo: band split + bitwise reassembly), the ncu launch list of the
# bench command and one `ncu --set full` capture of the solve kernel (CSV exports).
set -u
tag=${1:-r02}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_bench_2rank_1gpu.json 2> gpurun_out/${tag}_bench_2rank_1gpu.err
if [ "${NCU:-1}" = 1 ]; then
cmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$cmd > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv $cmd > gpurun_out/${tag}_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_solve_f32 -c 1 \
    -o /tmp/${tag}_solve $cmd > gpurun_out/${tag}_ncu_full.log 2>&1
if [ -f /tmp/${tag}_solve.ncu-rep ]; then
  cp /tmp/${tag}_solve.ncu-rep gpurun_out/
  ncu -i /tmp/${tag}_solve.ncu-rep --page details --csv > gpurun_out/${tag}_solve_details.csv
  ncu -i /tmp/${tag}_solve.ncu-rep --page raw --csv > gpurun_out/${tag}_solve_raw.csv
  ncu -i /tmp/${tag}_solve.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_solve_src.csv
fi
fi
ls -la gpurun_out | tail -20
