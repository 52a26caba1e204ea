cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-exposed --no-cpu --dims 2,1,1"
for k in 1 2; do
for v in head v1 v2; do
IGG_LIBRARY=$PWD/ab/libigg_$v.so timeout 600 $R > gpurun_out/ab_${v}_$k.log 2>&1
done
IGG_LIBRARY=$PWD/ab/libigg_v2.so timeout 600 $R --fused-mode 3 > gpurun_out/ab_v2m3_$k.log 2>&1
timeout 600 $R > gpurun_out/ab_new_$k.log 2>&1
done
echo done
