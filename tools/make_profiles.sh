#!/bin/bash
# Summaries of a tools/profile_round.sh capture into profiles/ (run here, after gpurun).
# usage: bash tools/make_profiles.sh TAG
TAG=${1:-r2}
O=gpurun_out
P=profiles
for f in bench_$TAG bench_${TAG}_reference bench_${TAG}_config4; do
  [ -s $O/$f.json ] && cp $O/$f.json $P/${f/bench_$TAG/${TAG}_bench}.json
done
cp $O/launches_$TAG.csv $P/${TAG}_launches.csv
python tools/launch_summary.py $O/launches_$TAG.csv $P/${TAG}_launches.txt > /dev/null
for wl in config5 config4; do
  n=16384; [ $wl = config4 ] && n=4096
  python tools/ncu_traffic.py $O/prof_${TAG}_$wl.ncu-rep nh_stream_kp $P/kp_traffic_$wl.json $wl $((4096*n)) > /dev/null
  for k in kp ks kc; do
    python tools/ncu_summary.py $O/prof_${TAG}_$wl.ncu-rep --kernel nh_stream_$k --source 25 \
        > $P/${TAG}_${wl}_${k}_ncu_summary.txt
  done
done
for f in kp_probe5 kp_probe4 kp_probe5g smoke; do
  [ -s $O/${f}_$TAG.txt ] && cp $O/${f}_$TAG.txt $P/${TAG}_$f.txt
done
ls -la $P | tail -30
