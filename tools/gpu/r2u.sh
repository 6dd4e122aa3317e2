set -x
mkdir -p gpurun_out
rm -f gpurun_out/ab_fuse.txt
for w in 1000 4000 8000; do
for f in 0 1; do
  r=$(NH_KP_FUSE_ADAPTIVE=$f timeout 900 python tools/kp_probe.py --workload config5 --members 2048 --warmup $w --steps 40 2>&1 | tail -1)
  echo "fuse$f warm$w $r" >> gpurun_out/ab_fuse.txt
done
done
for f in 0 1; do
  r=$(NH_KP_FUSE_ADAPTIVE=$f timeout 900 python tools/kp_probe.py --workload config4 --members 4096 --warmup 10000 --steps 40 2>&1 | tail -1)
  echo "fuse$f c4warm10000 $r" >> gpurun_out/ab_fuse.txt
done
NH_KP_FUSE_ADAPTIVE=1 timeout 900 python -m pytest tests/test_gpu_simulate.py tests/test_gpu_edges.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_fuse.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_fuse.txt
