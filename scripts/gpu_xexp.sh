cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/xf_*.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -s -k p2p > gpurun_out/xf_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/xf_pytest_multi.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed > gpurun_out/xf_n1.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-exposed --no-cpu --dims 2,1,1"
for m in 2 3 14 2 3; do
timeout 600 $R --fused-mode $m > gpurun_out/xf_m$m.log 2>&1
timeout 600 $R --fused-mode $m > gpurun_out/xf_m${m}b.log 2>&1
done
echo done
