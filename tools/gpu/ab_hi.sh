# A/B of library variants (gpurun_ab/<name>.so) on the probes at low and high flagged fraction,
# config 5 adaptive / global and config 4: usage ab_hi.sh name1 name2 ...
mkdir -p gpurun_out
out=gpurun_out/ab_hi_$(date +%s).txt
for rep in 1 2; do
  for v in "$@"; do
    for w in 1000 8000; do
      r=$(NH_LIB=gpurun_ab/$v.so timeout 900 python tools/kp_probe.py --workload config5 --members 2048 --warmup $w --steps 40 2>&1 | tail -1)
      echo "$v c5warm$w $r" >> $out
    done
    r=$(NH_LIB=gpurun_ab/$v.so timeout 900 python tools/kp_probe.py --workload config5 --members 2048 --warmup 200 --steps 40 --mode global 2>&1 | tail -1)
    echo "$v c5global $r" >> $out
    r=$(NH_LIB=gpurun_ab/$v.so timeout 900 python tools/kp_probe.py --workload config4 --members 4096 --warmup 200 --steps 40 2>&1 | tail -1)
    echo "$v c4 $r" >> $out
  done
done
cp $out gpurun_out/ab_hi_last.txt
