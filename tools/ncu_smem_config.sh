#!/bin/bash
# experiment: shared-memory configuration and L1 hit rate of k_solve_f32 per variant library
mkdir -p gpurun_out
for lib in "$@"; do
  TQSB_LIB=$PWD/paper_2205_02646_b200/$lib ncu --clock-control none -k regex:k_solve_f32 -c 1 \
    --metrics launch__shared_mem_config_size,launch__shared_mem_per_block_dynamic,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed \
    --csv python tools/variants.py --child --reps 1 --save /tmp/x.npy 2>/dev/null | grep -E '"(launch|l1tex|gpu__)' | awk -F'","' -v L=$lib '{print L, $(NF-2), $NF}'
done
