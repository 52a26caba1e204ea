cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/h37_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k binary32 > gpurun_out/h37_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h37_pytest.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dtype f32 --steps 100 --warmup 10"
timeout 600 $R > gpurun_out/h37_n2.log 2>&1
timeout 600 $R --no-e2e --fused-mode 16386 > gpurun_out/h37_n2_slabs.log 2>&1
timeout 600 $R --no-e2e --dims 1,2,1 > gpurun_out/h37_n2_y.log 2>&1
for f in h37_n2 h37_n2_slabs h37_n2_y; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/$f.log | head -1)" >> gpurun_out/h37_sum.txt; done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/h37_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/h37_pytest_multi.log
echo done
