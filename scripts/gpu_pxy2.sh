cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/xz_*
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed"
timeout 300 $B --periodic 1,1,0 --kc2 8 > gpurun_out/xz_pxy_k8.log 2>&1
timeout 300 $B --periodic 1,1,0 --kc2 16 > gpurun_out/xz_pxy_k16.log 2>&1
timeout 300 $B --periodic 1,1,1 --kc2 8 > gpurun_out/xz_pxyz_k8.log 2>&1
timeout 300 $B --periodic 1,0,1 --kc2 8 > gpurun_out/xz_pxz_k8.log 2>&1
timeout 300 $B --periodic 0,1,1 --kc2 8 > gpurun_out/xz_pyz_k8.log 2>&1
echo done
