cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/q6_*.log
timeout 1200 python -m pytest tests/test_gpu_heat.py tests/test_gpu_hide_comm.py tests/test_gpu_halo.py -x -q > gpurun_out/q6_pytest_single.log 2>&1; echo "rc=$?" >> gpurun_out/q6_pytest_single.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e --no-exposed"
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu > gpurun_out/q6_n1.log 2>&1
timeout 300 $R4 > gpurun_out/q6_n4.log 2>&1
timeout 300 $R4 --dims 1,2,2 > gpurun_out/q6_n4_122.log 2>&1
timeout 300 $R4 --dims 2,1,2 > gpurun_out/q6_n4_212.log 2>&1
timeout 300 $R4 --fused-mode 130 > gpurun_out/q6_n4_legacy.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/q6_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/q6_pytest_multi.log
echo done
