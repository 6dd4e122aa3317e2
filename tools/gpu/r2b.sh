mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_b.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_b.txt
timeout 300 python -m pytest tests/test_gpu_errors.py -m gpu -q -s > gpurun_out/pytest_errors_b.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_b.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_b.txt
