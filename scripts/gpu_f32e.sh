cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/h34_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k binary32 > gpurun_out/h34_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h34_pytest.log
B="python bench.py --dtype f32 --steps 100 --warmup 10 --no-cpu --no-e2e --no-exposed"
for v in 0 106 103 113 114 115 116 117 118 102 0 106 113; do
  timeout 300 $B --kernel $v > gpurun_out/h34_v$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/h34_v$v.log)" >> gpurun_out/h34_sweep.txt
done
H="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed --periodic 1,0,0"
for m in 2 4098 2 4098; do
  timeout 300 $H --fused-mode $m > gpurun_out/h34_px_m$m.log 2>&1
  echo "px m$m $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/h34_px_m$m.log)" >> gpurun_out/h34_sweep.txt
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dtype f32 --steps 100 --warmup 10"
timeout 600 $R > gpurun_out/h34_n2.log 2>&1
echo done
