set -x
mkdir -p gpurun_out
bash tools/gpu/ab.sh a2 a3 a3nohw a3nou
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_a3.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_a3.txt
timeout 900 python bench.py --cpu-steps 0 > gpurun_out/bench_a3.json 2> gpurun_out/bench_a3.err
