set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -q -x -k longer > gpurun_out/pytest_long.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_long.txt
