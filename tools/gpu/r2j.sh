set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_flux.py tests/test_gpu_errors.py -m gpu -q -x > gpurun_out/pytest_flux.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_flux.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2j.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2j.txt
