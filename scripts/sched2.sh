cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sched_*.log gpurun_out/bench2_*.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -k "not multi" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --timeline"
timeout 300 $B > gpurun_out/sched_A_full.log 2>&1
for sch in 0 1; do
timeout 300 $B --periodic 1,0,0 --bw 2,2,2 --xalign 1 --schedule $sch > gpurun_out/sched_s${sch}_bw2.log 2>&1
timeout 300 $B --periodic 1,0,0 --bw 16,2,2 --xalign 1 --schedule $sch > gpurun_out/sched_s${sch}_bw16_a1.log 2>&1
timeout 300 $B --periodic 1,0,0 --bw 16,2,2 --xalign 64 --schedule $sch > gpurun_out/sched_s${sch}_bw16_a64.log 2>&1
timeout 300 $B --periodic 1,1,1 --bw 2,2,2 --xalign 1 --schedule $sch > gpurun_out/sched_s${sch}_bw2_3ax.log 2>&1
done
for sch in 0 1; do
for path in nccl p2p; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus 2 --steps 100 --warmup 10 --path $path --no-e2e --bw 16,2,2 --xalign 1 --schedule $sch --timeline > gpurun_out/bench2_${path}_s${sch}.log 2>&1
done
done
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi.log
echo done
