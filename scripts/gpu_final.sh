cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/fin_*
timeout 600 python bench.py > gpurun_out/fin_n1.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/fin_n2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/fin_n4.log 2>&1
timeout 600 python bench.py --workload acoustic --steps 50 --warmup 5 > gpurun_out/fin_ac_n1.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fin_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/fin_pytest_gpu.log
echo done
