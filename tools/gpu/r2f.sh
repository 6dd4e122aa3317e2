set -x
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/host.txt 2>&1
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
timeout 600 python tools/kp_probe.py --workload config5 --members 4096 --warmup 1000 --steps 40 > gpurun_out/kp_probe5.txt 2>&1
timeout 600 python tools/kp_probe.py --workload config4 --members 4096 --warmup 200 --steps 40 > gpurun_out/kp_probe4.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nh_stream_kp --launch-skip 2 -c 1 -o gpurun_out/kp5 python tools/kp_probe.py --workload config5 --members 4096 --warmup 1000 --steps 4 > gpurun_out/ncu_kp5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nh_stream_kp --launch-skip 2 -c 1 -o gpurun_out/kp4 python tools/kp_probe.py --workload config4 --members 4096 --warmup 200 --steps 4 > gpurun_out/ncu_kp4.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
