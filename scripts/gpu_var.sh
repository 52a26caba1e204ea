cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/va_*.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --no-exposed --no-cpu"
for k in 1 2; do
for v in cur inl noinl lb9 stcs inl_lb9 inl_stcs; do
IGG_LIBRARY=$PWD/ab/libigg_$v.so timeout 300 $R --dims 2,1,1 > gpurun_out/va_${v}_$k.log 2>&1
done
done
IGG_LIBRARY=$PWD/ab/libigg_inl.so timeout 300 $R --dims 1,1,2 > gpurun_out/va_inl_z.log 2>&1
IGG_LIBRARY=$PWD/ab/libigg_inl.so timeout 300 $R --dims 1,2,1 > gpurun_out/va_inl_y.log 2>&1
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu"
IGG_LIBRARY=$PWD/ab/libigg_inl.so timeout 300 $B > gpurun_out/va_n1_default.log 2>&1
IGG_LIBRARY=$PWD/ab/libigg_inl.so timeout 300 $B --fused 2 > gpurun_out/va_n1_f2m2.log 2>&1
IGG_LIBRARY=$PWD/ab/libigg_inl.so timeout 300 $B --fused 2 --fused-mode 0 > gpurun_out/va_n1_f2m0.log 2>&1
IGG_LIBRARY=$PWD/ab/libigg_inl.so timeout 300 $B --fused 2 --skip-comm > gpurun_out/va_n1_f2skip.log 2>&1
IGG_LIBRARY=$PWD/ab/libigg_inl_stcs.so timeout 300 $B --fused 2 --skip-comm > gpurun_out/va_n1_f2skip_stcs.log 2>&1
echo done
