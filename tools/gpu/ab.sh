# A/B of library variants (gpurun_ab/<name>.so) on the K_P probe: usage ab.sh name1 name2 ...
mkdir -p gpurun_out
out=gpurun_out/ab_$(date +%s).txt
for rep in 1 2; do
  for v in "$@"; do
    for wl in config5 config4; do
      w=1000; [ $wl = config4 ] && w=200
      r=$(NH_LIB=gpurun_ab/$v.so timeout 600 python tools/kp_probe.py --workload $wl --members 4096 --warmup $w --steps 40 2>&1 | tail -1)
      echo "$v $wl $r" >> $out
    done
  done
done
cp $out gpurun_out/ab_last.txt
