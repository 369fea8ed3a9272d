#!/usr/bin/env bash
# BASELINE configs[3] (period sweep, 1 MP) and configs[4] (64-frame video, P = 16) on one B200.
tag=${1:-r01}
mkdir -p gpurun_out
for P in 4 8 16 32; do
  python bench.py --workload 1mp --period $P --steps 5 --warmup 3 > gpurun_out/${tag}_sweep_p$P.json 2> gpurun_out/${tag}_sweep_p$P.err
done
python bench.py --workload video --steps 3 --warmup 1 > gpurun_out/${tag}_video.json 2> gpurun_out/${tag}_video.err
tail -n 3 gpurun_out/${tag}_video.err
