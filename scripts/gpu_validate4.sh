cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/val_*.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/val_pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/val_pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/val_smoke.log
timeout 900 python bench.py > gpurun_out/val_n1.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/val_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/val_n4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29516 scripts/halo_sweep.py > gpurun_out/val_sweep4.log 2>&1
echo done
