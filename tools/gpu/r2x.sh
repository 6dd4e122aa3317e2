set -x
mkdir -p gpurun_out
rm -f gpurun_out/ab_tpf.txt
for rep in 1 2; do
for v in geo1b tpf; do
  for w in 1000 8000; do
    r=$(NH_LIB=gpurun_ab/$v.so timeout 900 python tools/kp_probe.py --workload config5 --members 2048 --warmup $w --steps 40 2>&1 | tail -1)
    echo "$v warm$w $r" >> gpurun_out/ab_tpf.txt
  done
  r=$(NH_LIB=gpurun_ab/$v.so timeout 900 python tools/kp_probe.py --workload config4 --members 4096 --warmup 200 --steps 40 2>&1 | tail -1)
  echo "$v c4 $r" >> gpurun_out/ab_tpf.txt
done
done
NH_LIB=gpurun_ab/tpf.so timeout 900 python -m pytest tests/test_gpu_simulate.py tests/test_gpu_edges.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_tpf.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_tpf.txt
