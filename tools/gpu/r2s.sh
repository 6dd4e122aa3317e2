set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -q -x -k threshold > gpurun_out/pytest_thr.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_thr.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2s.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2s.txt
