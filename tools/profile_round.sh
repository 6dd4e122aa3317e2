#!/bin/bash
# One GPU call: the driver's bench line (config 5), the reference arm, an ncu
# launch list of the same bench command and ncu --set full captures of the
# streaming kernels on the 4096-member probes (tools/kp_probe.py: the same
# per-cell work as the full ensemble; a full capture of a 26789-member block
# would replay 60 GB of state 40 times).
# usage (under gpurun): bash tools/profile_round.sh TAG
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
timeout 1500 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 900 python bench.py --impl reference > $O/bench_${TAG}_reference.json 2> $O/bench_${TAG}_reference.err
timeout 900 python bench.py --workload config4 --steps 2000 --cpu-steps 0 --global-steps 200 > $O/bench_${TAG}_config4.json 2> $O/bench_${TAG}_config4.err
# launch list of the bench command itself: the 1000 spin-up steps and 3 warm-up
# steps are 3 member blocks x 4 kernels each -> skip them, list 4 steps
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:nh_stream --launch-skip 12040 -c 96 --csv \
    --log-file $O/launches_$TAG.csv python bench.py --steps 8 --warmup 3 --cpu-steps 0 --no-e2e --global-steps 0 > $O/ncu_${TAG}_a.log 2>&1
for wl in config5 config4; do
  w=1000; [ $wl = config4 ] && w=200
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"nh_stream_k[psc]" --launch-skip $((w*3+1)) -c 4 \
      -o $O/prof_${TAG}_$wl python tools/kp_probe.py --workload $wl --members 4096 --warmup $w --steps 4 > $O/ncu_${TAG}_$wl.log 2>&1
done
timeout 600 python tools/kp_probe.py --workload config5 --members 4096 --warmup 1000 --steps 40 > $O/kp_probe5_$TAG.txt 2>&1
timeout 600 python tools/kp_probe.py --workload config4 --members 4096 --warmup 200 --steps 40 > $O/kp_probe4_$TAG.txt 2>&1
timeout 600 python tools/kp_probe.py --workload config5 --members 4096 --warmup 1000 --steps 40 --mode global > $O/kp_probe5g_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.txt 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.txt
