mkdir -p gpurun_out
OPENBLAS_NUM_THREADS=1 timeout 900 python tools/config3_margin.py > gpurun_out/config3_margin.txt 2>&1; echo "rc=$?" >> gpurun_out/config3_margin.txt
timeout 600 python -m pytest tests/test_gpu_capi_stub.py -m gpu -q > gpurun_out/pytest_stub.txt 2>&1
