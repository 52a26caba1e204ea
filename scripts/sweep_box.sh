cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sweep.log
timeout 600 python -m pytest tests/test_gpu_heat.py -x -q -m "gpu and not slow" -k variants > gpurun_out/pytest_heat.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_heat.log
for v in 20 50 51 52 53 54 55 56 20; do
  echo "variant $v" >> gpurun_out/sweep.log
  timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu --kernel $v >> gpurun_out/sweep.log 2>&1
done
echo done
