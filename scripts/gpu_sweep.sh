cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 scripts/halo_sweep.py > gpurun_out/sweep1e.log 2>&1
timeout 600 python -m pytest tests/test_gpu_halo.py -x -q > gpurun_out/small_pytest_halo.log 2>&1; echo "rc=$?" >> gpurun_out/small_pytest_halo.log
echo done
