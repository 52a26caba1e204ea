cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --timeline"
timeout 600 $R --path p2p --fused 1 > gpurun_out/fz_p2p_f1.log 2>&1
timeout 600 $R --path p2p --fused 1 --periodic 1,1,1 > gpurun_out/fz_p2p_f1_per3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s -k p2p > gpurun_out/pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi.log
echo done
