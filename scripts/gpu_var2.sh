cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/vb_*.log
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/vb_n1_default.log 2>&1
timeout 300 $B --fused 2 --skip-comm > gpurun_out/vb_n1_f2skip.log 2>&1
timeout 300 $B --fused 2 > gpurun_out/vb_n1_f2.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-exposed --no-cpu"
for k in 1 2; do
timeout 300 $R --dims 2,1,1 > gpurun_out/vb_x_$k.log 2>&1
timeout 300 $R --dims 2,1,1 --fused-mode 34 > gpurun_out/vb_x_m34_$k.log 2>&1
timeout 300 $R --dims 1,1,2 > gpurun_out/vb_z_$k.log 2>&1
timeout 300 $R --dims 1,1,2 --fused-mode 66 > gpurun_out/vb_z_m66_$k.log 2>&1
timeout 300 $R --dims 1,1,2 --fused-mode 34 > gpurun_out/vb_z_m34_$k.log 2>&1
timeout 300 $R --dims 2,1,1 --fused-mode 14 > gpurun_out/vb_x_m14_$k.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s -k p2p > gpurun_out/vb_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/vb_pytest_multi.log
echo done
