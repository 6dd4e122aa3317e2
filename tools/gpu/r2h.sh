set -x
mkdir -p gpurun_out
./tools/fp64_peak/fp64_peak > gpurun_out/fp64_peak.json 2> gpurun_out/fp64_peak.err
bash tools/gpu/ab.sh all a2 a2nocrit a2noexp2 a2nod0 t256 t192 t96
for v in a2 a2nod0 t256; do
NH_LIB=gpurun_ab/$v.so timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$v.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$v.txt
done
