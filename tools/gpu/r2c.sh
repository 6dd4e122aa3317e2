mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_capi_stub.py tests/test_reference_objects.py -m gpu -q -s -k "config3 or stub or reference_objects or full_length" > gpurun_out/pytest_c3.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c3.txt
