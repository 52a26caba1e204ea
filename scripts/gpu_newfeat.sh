cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hide_comm.py tests/test_gpu_halo.py -x -q > gpurun_out/nf_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/nf_pytest.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/nf_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/nf_pytest_multi.log
echo done
