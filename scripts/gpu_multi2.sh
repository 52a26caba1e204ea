cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/bench2_*.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for bw in 16,2,2 2,2,2; do
for path in nccl p2p; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus 2 --steps 100 --warmup 10 --path $path --no-e2e --bw $bw > gpurun_out/bench2_${path}_$bw.log 2>&1
done
done
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu > gpurun_out/bench1.log 2>&1
echo done
