set -x
mkdir -p gpurun_out
for p in 0 8 16 32; do
for wl in config5 config4; do
  w=1000; [ $wl = config4 ] && w=200
  r=$(NH_KP_PERSIST=$p timeout 600 python tools/kp_probe.py --workload $wl --members 4096 --warmup $w --steps 40 2>&1 | tail -1)
  echo "persist$p $wl $r" >> gpurun_out/ab_persist.txt
done
done
NH_KP_PERSIST=8 timeout 900 python -m pytest tests/test_gpu_simulate.py tests/test_gpu_edges.py -m gpu -q -x > gpurun_out/pytest_persist.txt 2>&1
