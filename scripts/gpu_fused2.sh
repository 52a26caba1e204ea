cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/fz_*.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --fused 2 > gpurun_out/fz_1gpu_f2.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --timeline"
timeout 600 $R --path p2p --fused 1 > gpurun_out/fz_p2p_f1.log 2>&1
timeout 600 $R --path p2p --fused 1 --skip-comm > gpurun_out/fz_p2p_f1_nocomm.log 2>&1
timeout 600 $R --path p2p --fused 1 --periodic 1,0,0 > gpurun_out/fz_p2p_f1_perx.log 2>&1
timeout 600 $R --path p2p --fused 1 --periodic 1,1,1 > gpurun_out/fz_p2p_f1_per3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s -k p2p > gpurun_out/pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi.log
echo done
