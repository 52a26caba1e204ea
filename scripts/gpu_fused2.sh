cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/fm_*.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --timeline --no-exposed"
for m in 0 1 2 3; do
timeout 600 $R --path p2p --fused 1 --fused-mode $m > gpurun_out/fm_f1_m$m.log 2>&1
timeout 600 $R --path p2p --fused 1 --fused-mode $m --skip-comm > gpurun_out/fm_nocomm_m$m.log 2>&1
done
echo done
