set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_members.py > gpurun_out/pytest_gpu_r2m.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2m.txt
timeout 900 python bench.py --cpu-steps 0 > gpurun_out/bench_r2m.json 2> gpurun_out/bench_r2m.err
NH_KFIN_LIST=0 timeout 900 python bench.py --cpu-steps 0 --no-e2e --global-steps 0 > gpurun_out/bench_r2m_nofin.json 2> gpurun_out/bench_r2m_nofin.err
timeout 600 python tools/kp_probe.py --workload config5 --members 4096 --warmup 1000 --steps 40 > gpurun_out/kp_probe5_r2m.txt 2>&1
