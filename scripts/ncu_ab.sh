cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --fused 2 > gpurun_out/ab_f2_timing.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu > gpurun_out/ab_v20_timing.log 2>&1
timeout 300 $B --fused 2 > gpurun_out/ab_f2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:heat_fused -s 3 -c 1 -o gpurun_out/prof_f2b $B --fused 2 > gpurun_out/ncu_f2b.log 2>&1
echo done
