cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/xb_*
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k "self_wrap" > gpurun_out/xb_pytest_self.log 2>&1; echo "rc=$?" >> gpurun_out/xb_pytest_self.log
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed"
timeout 300 $B > gpurun_out/xb_n1.log 2>&1
timeout 300 $B --periodic 1,0,0 > gpurun_out/xb_px.log 2>&1
timeout 300 $B --periodic 1,0,0 --fused-mode 2050 > gpurun_out/xb_px_old.log 2>&1
timeout 300 $B --periodic 1,1,1 > gpurun_out/xb_pxyz.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed"
timeout 300 $R > gpurun_out/xb_x.log 2>&1
timeout 300 $R --fused-mode 2050 > gpurun_out/xb_x_old.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s -k p2p > gpurun_out/xb_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/xb_pytest_multi.log
echo done
