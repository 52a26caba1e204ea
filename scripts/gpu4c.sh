cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/q5_*.log
timeout 300 python bench.py --steps 100 --warmup 10 > gpurun_out/q5_n1.log 2>&1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10"
timeout 400 $R2 > gpurun_out/q5_n2.log 2>&1
timeout 400 $R4 > gpurun_out/q5_n4.log 2>&1
timeout 300 $R4 --no-e2e --no-exposed --dims 1,2,2 > gpurun_out/q5_n4_122.log 2>&1
timeout 300 $R4 --no-e2e --no-exposed --dims 2,1,2 > gpurun_out/q5_n4_212.log 2>&1
timeout 300 $R4 --no-e2e --no-exposed --dims 1,1,4 > gpurun_out/q5_n4_114.log 2>&1
timeout 300 $R4 --no-e2e --no-exposed --dims 4,1,1 > gpurun_out/q5_n4_411.log 2>&1
timeout 300 $R4 --no-e2e --no-exposed --per-step > gpurun_out/q5_n4_ps.log 2>&1
timeout 300 $R4 --no-e2e --no-exposed --fused-mode 130 > gpurun_out/q5_n4_legacy.log 2>&1
timeout 300 $R4 --no-e2e --no-exposed --path nccl > gpurun_out/q5_n4_nccl.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/q5_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/q5_pytest_multi.log
echo done
