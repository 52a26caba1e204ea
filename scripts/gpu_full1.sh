cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "not multi" > gpurun_out/full1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/full1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full1_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/full1_smoke.log
timeout 900 python bench.py > gpurun_out/full1_bench.log 2>&1
echo done
