#!/bin/bash
# Summaries of a tools/profile_round.sh capture into profiles/ (run here, after gpurun).
# usage: bash tools/make_profiles.sh TAG
TAG=${1:-r1}
O=gpurun_out
P=profiles
cp $O/bench_$TAG.json $P/${TAG}_bench.json
cp $O/bench_${TAG}_global.json $P/${TAG}_bench_global.json
cp $O/launches_$TAG.csv $P/${TAG}_launches.csv
python tools/launch_summary.py $O/launches_$TAG.csv $P/${TAG}_launches.txt > /dev/null
python tools/ncu_traffic.py $O/prof_$TAG.ncu-rep nh_stream_kp $P/kp_traffic.json > /dev/null
for k in kp ks kc; do
  python tools/ncu_summary.py $O/prof_$TAG.ncu-rep --kernel nh_stream_$k --source 25 \
      > $P/${TAG}_${k}_ncu_summary.txt
done
ls -la $P
