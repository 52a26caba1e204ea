cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/fn3_*
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/fn3_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/fn3_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as G; G.smoke(); print('SMOKE OK')" > gpurun_out/fn3_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/fn3_n1.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fn3_ref.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2"
timeout 300 $R > gpurun_out/fn3_n2.log 2>&1
echo done
