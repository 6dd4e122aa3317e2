set -x
O=gpurun_out; TAG=${1:-r2a}
for wl in config5 config4; do
  w=1000; [ $wl = config4 ] && w=200
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"nh_stream_k[psc]" --launch-skip $((w*3+1)) -c 4 \
      -o $O/prof_${TAG}_$wl python tools/kp_probe.py --workload $wl --members 4096 --warmup $w --steps 4 > $O/ncu_${TAG}_$wl.log 2>&1
done
