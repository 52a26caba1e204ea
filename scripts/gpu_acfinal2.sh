cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/acf2_*
timeout 110 python -m pytest tests/test_gpu_multi.py -k "parity and p2p" -x -q > gpurun_out/acf2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/acf2_pytest.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2"
timeout 50 $R --workload acoustic --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/acf2_bench_n2.log 2>&1
echo done
