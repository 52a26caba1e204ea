cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/fy_*.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --fused 2 > gpurun_out/fy_1gpu_f2.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu > gpurun_out/fy_1gpu.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e"
timeout 600 $R > gpurun_out/fy_2gpu.log 2>&1
timeout 600 $R --timeline --no-exposed > gpurun_out/fy_2gpu_tl.log 2>&1
timeout 600 $R --skip-comm > gpurun_out/fy_2gpu_nocomm.log 2>&1
echo done
