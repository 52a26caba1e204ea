cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu" -x -q -k "not multi" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_box -s 2 -c 1 -o gpurun_out/prof_box $B > gpurun_out/ncu_full.log 2>&1
echo done
