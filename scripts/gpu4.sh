cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/g4z_*.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/g4z_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/g4z_pytest_multi.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e"
timeout 900 $R4 > gpurun_out/g4z_fused4.log 2>&1
timeout 900 $R4 --skip-comm > gpurun_out/g4z_fused4_nocomm.log 2>&1
timeout 900 $R4 --fused 0 > gpurun_out/g4z_split4.log 2>&1
timeout 900 $R4 --path nccl > gpurun_out/g4z_nccl4.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --fused 2 > gpurun_out/g4z_1gpu_f2.log 2>&1
echo done
