#!/usr/bin/env bash
# one GPU call's worth of round evidence: headline bench + reference arm + ncu captures
# (tools/profile_round.sh), the period sweep and video stream (tools/sweep.sh), and the
# L-JSDE baseline comparison (tools/ljsde_bench.py)
tag=${1:-r01}
bash tools/profile_round.sh $tag
bash tools/sweep.sh $tag
python tools/ljsde_bench.py > gpurun_out/${tag}_ljsde.json 2> gpurun_out/${tag}_ljsde.err
