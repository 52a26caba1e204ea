cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/fs2_*
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -s -k full_size > gpurun_out/fs2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fs2_pytest.log
echo done
