set -x
mkdir -p gpurun_out
timeout 1500 python tools/full_length.py --workload config5 --mode adaptive > gpurun_out/full_config5_adaptive.json 2> gpurun_out/full_config5_adaptive.err
timeout 900 python tools/full_length.py --workload config5 --mode global --steps 2000 > gpurun_out/full_config5_global2000.json 2> gpurun_out/full_config5_global.err
timeout 600 python tools/full_length.py --workload config4 --mode adaptive > gpurun_out/full_config4_adaptive.json 2> gpurun_out/full_config4_adaptive.err
timeout 600 python -m pytest tests/test_gpu_simulate.py -m gpu -q -x > gpurun_out/pytest_sim.txt 2>&1
