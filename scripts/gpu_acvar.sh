cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/av_*
B="python bench.py --workload acoustic --steps 30 --warmup 5 --no-cpu --no-e2e"
for k in 1 2; do
for v in cur ac_4_16 ac_4_64 ac_8_32 ac_8_64 ac_2_64 ac_4_128; do
  if [ $v = cur ]; then L=""; else L="IGG_LIBRARY=$PWD/ab/libigg_$v.so"; fi
  env $L timeout 120 $B > gpurun_out/av_${v}_$k.log 2>&1
  echo "$v $k $(python scripts/show_ac.py gpurun_out/av_${v}_$k.log)" >> gpurun_out/av_summary.txt
done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/av_launches.csv $B --steps 5 --warmup 3 > gpurun_out/av_ncu_list.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:acoustic -c 2 --csv --page raw --log-file gpurun_out/av_ncu_full.csv python bench.py --workload acoustic --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/av_ncu_full.log 2>&1
echo done
