cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/v4_*.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e --no-exposed"
timeout 900 $R4 > gpurun_out/v4_fused.log 2>&1
timeout 900 $R4 --skip-comm > gpurun_out/v4_nocomm.log 2>&1
timeout 900 $R4 --skip-comm --kc2 8 > gpurun_out/v4_nocomm_k8.log 2>&1
timeout 900 $R4 --fused 0 --skip-comm > gpurun_out/v4_split_nocomm.log 2>&1
for d in 0 1 2 3; do CUDA_VISIBLE_DEVICES=$d timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu > gpurun_out/v4_gpu$d.log 2>&1; done
echo done
