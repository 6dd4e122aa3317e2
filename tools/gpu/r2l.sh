set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests/test_gpu_members.py -m gpu -q -s --durations=5 > gpurun_out/pytest_members.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_members.txt
for blk in 512 1024 2048; do
timeout 900 python bench.py --cpu-steps 0 --global-steps 0 --e2e-block $blk > gpurun_out/bench_e2e_$blk.json 2> gpurun_out/bench_e2e_$blk.err
done
timeout 600 python tools/kp_probe.py --workload config5 --members 4096 --warmup 1000 --steps 40 > gpurun_out/kp_probe5_kc.txt 2>&1
timeout 600 python tools/kp_probe.py --workload config4 --members 4096 --warmup 200 --steps 40 > gpurun_out/kp_probe4_kc.txt 2>&1
