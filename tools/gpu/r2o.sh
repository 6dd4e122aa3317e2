set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests/test_gpu_members.py -m gpu -q -s > gpurun_out/pytest_members2.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_members2.txt
