cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r01_bench_default.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/r01_bench_reference.log 2>&1
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/r01_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $B > gpurun_out/r01_ncu_launch.log 2>&1
timeout 300 $B > gpurun_out/r01_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_box_async -s 3 -c 1 -o gpurun_out/r01_prof_stencil $B > gpurun_out/r01_ncu_full.log 2>&1
echo done
