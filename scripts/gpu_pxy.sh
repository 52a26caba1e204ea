cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/xy_*
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed"
timeout 300 $B --periodic 1,1,0 > gpurun_out/xy_pxy.log 2>&1
timeout 300 $B --periodic 1,0,0 > gpurun_out/xy_px.log 2>&1
timeout 300 $B --periodic 1,0,1 > gpurun_out/xy_pxz.log 2>&1
S="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-exposed --periodic 1,1,0"
timeout 300 $S > gpurun_out/xy_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_fused -s 6 -c 1 -o gpurun_out/xy_pxy $S > gpurun_out/xy_ncu.log 2>&1
echo done
