cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/nd_*.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e --no-exposed"
for k in 8 16; do timeout 900 $R4 --kc2 $k > gpurun_out/nd4_k$k.log 2>&1; done
timeout 900 $R4 --kc2 8 --timeline > gpurun_out/nd4_k8_tl.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-exposed"
timeout 600 $R > gpurun_out/nd2.log 2>&1
echo done
