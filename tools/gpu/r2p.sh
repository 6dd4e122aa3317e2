set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_golden.py -m gpu -q -s -k "config3 or full_length" > gpurun_out/pytest_c3.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c3.txt
OPENBLAS_NUM_THREADS=1 timeout 1500 python tools/config3_margin.py > gpurun_out/config3_margin.txt 2>&1; echo "rc=$?" >> gpurun_out/config3_margin.txt
