cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/h36_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k binary32 > gpurun_out/h36_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h36_pytest.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dtype f32 --steps 100 --warmup 10 --no-e2e"
for x in 64 1 64 1; do
  timeout 600 $R --xalign $x > gpurun_out/h36_n2_xa$x.log 2>&1
  echo "xa$x $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/h36_n2_xa$x.log) $(grep -o '"exposed_halo": {[^}]*}' gpurun_out/h36_n2_xa$x.log)" >> gpurun_out/h36_sweep.txt
done
for d in 1,2,1 1,1,2; do
  timeout 600 $R --dims $d > gpurun_out/h36_n2_d$d.log 2>&1
  echo "dims$d $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/h36_n2_d$d.log) $(grep -o '"exposed_halo": {[^}]*}' gpurun_out/h36_n2_d$d.log)" >> gpurun_out/h36_sweep.txt
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/h36_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/h36_pytest_multi.log
echo done
