cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ae_*.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -s -k p2p > gpurun_out/ae_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/ae_pytest_multi.log
for d in 2,1,1 1,2,1 1,1,2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-exposed --dims $d > gpurun_out/ae_$d.log 2>&1
done
echo done
