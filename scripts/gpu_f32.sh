cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/f32_*
timeout 1200 python -m pytest tests/test_gpu_heat.py tests/test_gpu_halo.py tests/test_gpu_hide_comm.py tests/test_gpu_acoustic.py -x -q > gpurun_out/f32_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f32_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/f32_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/f32_pytest_multi.log
echo done
