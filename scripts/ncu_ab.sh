cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/prof_fz3.ncu-rep
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --fused 2"
timeout 300 $B > gpurun_out/ab_f2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:heat_fused -s 3 -c 1 -o gpurun_out/prof_fz3 $B > gpurun_out/ncu_fz3.log 2>&1
echo done
