# One GPU call that re-checks a tree: the GPU suite, smoke(), the driver's
# bench line and the reference arm.  usage (under gpurun): bash tools/gpu/verify.sh TAG
TAG=${1:-check}
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.txt
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err
