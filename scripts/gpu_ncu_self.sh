cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/nc_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k self_wrap > gpurun_out/nc_pytest_self.log 2>&1; echo "rc=$?" >> gpurun_out/nc_pytest_self.log
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-exposed"
for v in "f2:--fused 2" "px:--periodic 1,0,0" "py:--periodic 0,1,0" "pxpush:--periodic 1,0,0 --fused-mode 258"; do
  name=${v%%:*}; args=${v#*:}
  timeout 300 $B $args > gpurun_out/nc_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_fused -s 6 -c 1 -o gpurun_out/nc_$name $B $args > gpurun_out/nc_ncu_$name.log 2>&1
done
echo done
