cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/g4_*.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -s -k p2p > gpurun_out/g4_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/g4_pytest_multi.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10 --timeline --no-e2e"
timeout 900 $R4 > gpurun_out/g4_bench4_fused.log 2>&1
timeout 900 $R4 --fused 0 > gpurun_out/g4_bench4_split.log 2>&1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 100 --warmup 10 --timeline --no-e2e"
timeout 900 $R2 > gpurun_out/g4_bench2_fused.log 2>&1
timeout 900 $R2 --skip-comm > gpurun_out/g4_bench2_fused_nocomm.log 2>&1
echo done
