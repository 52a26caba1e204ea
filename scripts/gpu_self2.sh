cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sw_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k self_wrap > gpurun_out/sw_pytest_self.log 2>&1; echo "rc=$?" >> gpurun_out/sw_pytest_self.log
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed"
timeout 300 $B > gpurun_out/sw_n1.log 2>&1
timeout 300 $B --fused 2 > gpurun_out/sw_f2.log 2>&1
timeout 300 $B --periodic 0,1,0 > gpurun_out/sw_py.log 2>&1
timeout 300 $B --periodic 0,1,0 --per-step > gpurun_out/sw_py_ps.log 2>&1
timeout 300 $B --periodic 0,0,1 > gpurun_out/sw_pz.log 2>&1
timeout 300 $B --periodic 1,0,0 > gpurun_out/sw_px.log 2>&1
timeout 300 $B --periodic 1,0,0 --fused-mode 258 > gpurun_out/sw_px_push.log 2>&1
S="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-exposed --periodic 0,1,0"
timeout 300 $S > gpurun_out/sw_plain_py.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sw_launches_py.csv $S > gpurun_out/sw_ncu_py.log 2>&1
echo done
