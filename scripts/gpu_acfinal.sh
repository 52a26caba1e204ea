cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/acf_*
timeout 200 python -m pytest tests/test_gpu_acoustic.py tests/test_gpu_hide_comm.py -x -q > gpurun_out/acf_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/acf_pytest.log
timeout 120 python bench.py --workload acoustic --steps 50 --warmup 5 > gpurun_out/acf_bench_n1.log 2>&1
timeout 120 python -c "import __graft_entry__ as G; G.smoke(); print('SMOKE OK')" > gpurun_out/acf_smoke.log 2>&1
echo done
