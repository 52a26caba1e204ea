cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/g32_*
timeout 600 python bench.py --dtype f32 --steps 100 --warmup 10 > gpurun_out/g32_n1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dtype f32 --steps 100 --warmup 10 > gpurun_out/g32_n2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s > gpurun_out/g32_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/g32_pytest_multi.log
echo done
