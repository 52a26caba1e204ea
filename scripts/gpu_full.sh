cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/fz_*
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/fz_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/fz_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/fz_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fz_smoke.log
echo done
