cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/q7_*.log
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q -k "self_wrap or low_dim" > gpurun_out/q7_pytest_self.log 2>&1; echo "rc=$?" >> gpurun_out/q7_pytest_self.log
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-exposed"
timeout 300 $B > gpurun_out/q7_n1.log 2>&1
timeout 300 $B --periodic 1,1,0 > gpurun_out/q7_pxy.log 2>&1
timeout 300 $B --periodic 1,1,1 > gpurun_out/q7_pxyz.log 2>&1
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-exposed"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e --no-exposed"
timeout 300 $R2 > gpurun_out/q7_n2.log 2>&1
timeout 300 $R4 > gpurun_out/q7_n4.log 2>&1
timeout 300 $R4 --dims 1,2,2 > gpurun_out/q7_n4_122.log 2>&1
timeout 300 $R4 --dims 2,1,2 > gpurun_out/q7_n4_212.log 2>&1
timeout 300 $R4 --per-step > gpurun_out/q7_n4_ps.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/q7_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/q7_pytest_multi.log
echo done
