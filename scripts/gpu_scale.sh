cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sc_*.log
timeout 900 python bench.py > gpurun_out/sc_n1.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/sc_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/sc_n4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --path nccl > gpurun_out/sc_n4_nccl.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --path nccl > gpurun_out/sc_n2_nccl.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/sc_ref_n1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 4 --impl reference > gpurun_out/sc_ref_n4.log 2>&1
echo done
