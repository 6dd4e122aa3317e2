set -x
mkdir -p gpurun_out
bash tools/gpu/ab.sh geo0 geo1
NH_LIB=gpurun_ab/geo1.so timeout 900 python -m pytest tests/test_gpu_simulate.py tests/test_gpu_edges.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_geo.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_geo.txt
