cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ac_*.log
timeout 900 python -m pytest tests/test_gpu_acoustic.py -x -q > gpurun_out/ac_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ac_pytest.log
timeout 300 python bench.py --workload acoustic --steps 50 --warmup 5 > gpurun_out/ac_bench_n1.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu > gpurun_out/ac_heat_n1.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-exposed --no-cpu"
for k in 1 2; do
IGG_LIBRARY=$PWD/ab/libigg_head.so timeout 600 $R --dims 2,1,1 > gpurun_out/ac_head_$k.log 2>&1
timeout 600 $R --dims 2,1,1 > gpurun_out/ac_new_$k.log 2>&1
done
timeout 600 $R --workload acoustic --steps 50 > gpurun_out/ac_bench_n2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/ac_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/ac_pytest_multi.log
echo done
