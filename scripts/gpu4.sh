cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/g4y_*.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -s -k p2p > gpurun_out/g4y_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/g4y_pytest_multi.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10 --timeline --no-e2e --no-exposed"
timeout 900 $R4 --fused 1 > gpurun_out/g4y_fused.log 2>&1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 100 --warmup 10 --timeline --no-e2e --no-exposed"
timeout 900 $R2 --fused 1 > gpurun_out/g4y_fused2.log 2>&1
echo done
