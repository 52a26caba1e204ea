cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/h35_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k binary32 > gpurun_out/h35_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h35_pytest.log
B="python bench.py --dtype f32 --steps 100 --warmup 10 --no-cpu --no-e2e --no-exposed"
for v in 0 100 113 119 120 121 122 123 124 125 126 0 100; do
  timeout 300 $B --kernel $v > gpurun_out/h35_v$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/h35_v$v.log)" >> gpurun_out/h35_sweep.txt
done
timeout 600 python bench.py --dtype f32 --steps 100 --warmup 10 > gpurun_out/h35_n1.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dtype f32 --steps 100 --warmup 10"
timeout 600 $R > gpurun_out/h35_n2.log 2>&1
timeout 600 $R --timeline --no-exposed > gpurun_out/h35_n2_tl.log 2>&1
B="python bench.py --dtype f32 --steps 5 --warmup 3 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h35_launches.csv $B > gpurun_out/h35_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_f32_async -s 3 -c 1 -o gpurun_out/h35_prof $B > gpurun_out/h35_ncu_full.log 2>&1
echo done
