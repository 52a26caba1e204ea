cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/xw_*
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed --periodic 1,1,0"
timeout 300 $B > gpurun_out/xw_pxy.log 2>&1
timeout 300 $B --fused-mode 514 > gpurun_out/xw_pxy_nofwd.log 2>&1
timeout 300 $B --fused-mode 6 > gpurun_out/xw_pxy_norecv.log 2>&1
timeout 300 $B --kc2 32 > gpurun_out/xw_pxy_k32.log 2>&1
echo done
