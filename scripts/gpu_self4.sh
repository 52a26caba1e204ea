cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sx_*
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed"
timeout 300 $B > gpurun_out/sx_n1.log 2>&1
timeout 300 $B --periodic 1,0,0 > gpurun_out/sx_px.log 2>&1
timeout 300 $B --periodic 1,0,0 --fused-mode 34 > gpurun_out/sx_px_m34.log 2>&1
timeout 300 $B --periodic 1,0,0 --fused-mode 35 > gpurun_out/sx_px_m35.log 2>&1
timeout 300 $B --periodic 0,0,1 --fused-mode 34 > gpurun_out/sx_pz_m34.log 2>&1
timeout 300 $B --periodic 0,1,0 --fused-mode 34 > gpurun_out/sx_py_m34.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed"
timeout 300 $R --dims 2,1,1 > gpurun_out/sx_x.log 2>&1
timeout 300 $R --dims 2,1,1 --fused-mode 34 > gpurun_out/sx_x_m34.log 2>&1
echo done
