cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/k2_*.log
for k in 4 8 16 32; do timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --fused 2 --kc2 $k > gpurun_out/k2_f2_$k.log 2>&1; done
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu > gpurun_out/k2_v20.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --fused 2 --fused-mode 0 > gpurun_out/k2_f2_m0.log 2>&1
echo done
