set -x
mkdir -p gpurun_out
bash tools/gpu/ab.sh base mm d0 ec all
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py --cpu-steps 0 --global-steps 0 > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_probe.py > gpurun_out/sanitize_$t.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$t.txt
done
