# ncu --set full of k_solve_f32 for several library variants (1 MP, one launch each);
# exports the raw and per-instruction source pages as CSV and drops the reports.
set -e
for v in "$@"; do
  lib=$PWD/paper_2205_02646_b200/libtqsb_$v.so
  [ "$v" = base ] && lib=$PWD/paper_2205_02646_b200/libtqsb.so
  TQSB_LIB=$lib python tools/prof_solve.py --reps 1 > gpurun_out/plain_$v.log 2>&1
  TQSB_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:${KREG:-k_solve} -c 1 -o /tmp/prof_$v python tools/prof_solve.py --reps 1 > gpurun_out/ncu_$v.log 2>&1
  ncu -i /tmp/prof_$v.ncu-rep --page raw --csv > gpurun_out/raw_$v.csv
  ncu -i /tmp/prof_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$v.csv
  ncu -i /tmp/prof_$v.ncu-rep --page details --csv > gpurun_out/details_$v.csv
done
