set -x
mkdir -p gpurun_out
for blk in 2048 4096 8192; do
timeout 900 python bench.py --cpu-steps 0 --global-steps 0 --e2e-block $blk > gpurun_out/bench_e2e_$blk.json 2> gpurun_out/bench_e2e_$blk.err
done
