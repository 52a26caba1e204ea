cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/h32_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k binary32 > gpurun_out/h32_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h32_pytest.log
timeout 600 python bench.py --dtype f32 --steps 100 --warmup 10 > gpurun_out/h32_n1.log 2>&1
B="python bench.py --dtype f32 --steps 5 --warmup 3 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h32_launches.csv $B > gpurun_out/h32_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_f32_async -s 3 -c 1 -o gpurun_out/h32_prof $B > gpurun_out/h32_ncu_full.log 2>&1
echo done
