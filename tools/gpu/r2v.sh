set -x
mkdir -p gpurun_out
rm -f gpurun_out/ab_ks.txt
for v in default ks9 ks10; do
  lib=gpurun_ab/$v.so; [ $v = default ] && lib=paper_2505_17025_b200/_lib/libnhswe_b200.so
  for w in 1000 8000; do
    r=$(NH_LIB=$lib timeout 900 python tools/kp_probe.py --workload config5 --members 2048 --warmup $w --steps 40 2>&1 | tail -1)
    echo "$v warm$w $r" >> gpurun_out/ab_ks.txt
  done
done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2v.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2v.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2v.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r2v.txt
