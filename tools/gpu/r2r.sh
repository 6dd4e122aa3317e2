set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_simulate.py -m gpu -q -x -k advance_host > gpurun_out/pytest_host.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_host.txt
timeout 900 python bench.py --cpu-steps 0 --global-steps 0 > gpurun_out/bench_r2r.json 2> gpurun_out/bench_r2r.err
