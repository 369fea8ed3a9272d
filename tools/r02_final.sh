#!/usr/bin/env bash
# End-of-round evidence on one B200 (under gpurun): GPU suite, smoke, the bench line
# (default flags, as the driver runs it), the reference arm, the period sweep
# (configs[3]) and the 64-frame video (configs[4]), then the ncu launch list.
set -u
tag=${1:-r02f}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
tail -2 gpurun_out/${tag}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
cat gpurun_out/${tag}_smoke.log
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2>&1
for P in 4 8 16 32; do
  python bench.py --workload 1mp --period $P --steps 5 --warmup 3 --no-cpu-baseline \
      > gpurun_out/${tag}_sweep_p$P.json 2> gpurun_out/${tag}_sweep_p$P.err
done
python bench.py --workload video --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_video.json 2> gpurun_out/${tag}_video.err
if [ "${NCU:-1}" = 1 ]; then
  cmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe"
  $cmd > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_launches.csv $cmd > gpurun_out/${tag}_ncu_list.log 2>&1
fi
ls gpurun_out | grep ${tag}
