cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/h33_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k binary32 > gpurun_out/h33_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h33_pytest.log
B="python bench.py --dtype f32 --steps 100 --warmup 10 --no-cpu --no-e2e --no-exposed"
for v in 0 101 102 103 104 105 106 107 108 109 110 111 112 0; do
  timeout 300 $B --kernel $v > gpurun_out/h33_v$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/h33_v$v.log)" >> gpurun_out/h33_sweep.txt
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/h33_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/h33_pytest_multi.log
echo done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dtype f32 --steps 100 --warmup 10 > gpurun_out/h33_n2.log 2>&1
echo done2
