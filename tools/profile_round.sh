#!/bin/bash
# One GPU call: bench line, launch list and ncu --set full of the streaming kernels.
# usage (under gpurun): bash tools/profile_round.sh TAG
set -e
TAG=${1:-r1}
O=gpurun_out
python bench.py > $O/bench_$TAG.log 2>&1
tail -1 $O/bench_$TAG.log > $O/bench_$TAG.json
python bench.py --mode global --steps 500 --cpu-steps 0 --no-e2e 2>&1 | tail -1 > $O/bench_${TAG}_global.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:nh_ -c 60 --csv \
    --log-file $O/launches_$TAG.csv python bench.py --steps 8 --warmup 3 --cpu-steps 0 --no-e2e > $O/ncu_${TAG}_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"nh_stream_k[psc]" --launch-skip 12 -c 3 \
    -o $O/prof_$TAG python bench.py --steps 8 --warmup 3 --cpu-steps 0 --no-e2e > $O/ncu_${TAG}_b.log 2>&1
