cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/av2_*
B="python bench.py --workload acoustic --steps 30 --warmup 5 --no-cpu --no-e2e"
V="cur ac_4_16 ac_4_8 ac_8_16 ac_8_8 ac_2_16 ac_4_12"
for k in 1 2; do
for v in $V; do
  if [ $v = cur ]; then L=""; else L="IGG_LIBRARY=$PWD/ab/libigg_$v.so"; fi
  env $L timeout 120 $B > gpurun_out/av2_${v}_$k.log 2>&1
  echo "$v $k $(python scripts/show_ac.py gpurun_out/av2_${v}_$k.log)" >> gpurun_out/av2_summary.txt
done
done
for v in ac_4_16 ac_4_8 ac_8_16 ac_8_8 ac_2_16 ac_4_12; do
  env IGG_LIBRARY=$PWD/ab/libigg_$v.so timeout 150 python -m pytest tests/test_gpu_acoustic.py -x -q > gpurun_out/av2_pytest_$v.log 2>&1
  echo "parity $v rc=$? $(tail -1 gpurun_out/av2_pytest_$v.log)" >> gpurun_out/av2_summary.txt
done
echo done
