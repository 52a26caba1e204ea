# 2-GPU validation and measurements (gpurun --gpus 2): tests, bench 2x1x1 / 1x2x1 / 1x1x2, halo sweep, B:10
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; T=${TAG:-m2}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29519 --nproc-per-node 2"
timeout 1500 python -m pytest tests -q -m gpu -k "multi" > gpurun_out/${T}_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_multi.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/${T}_n1.json 2> gpurun_out/${T}_n1.err
for d in 2,1,1 1,2,1 1,1,2; do
  timeout 600 $TR bench.py --gpus 2 --dims $d --no-e2e > gpurun_out/${T}_n2_${d//,/}.json 2> gpurun_out/${T}_n2_${d//,/}.err
done
timeout 600 $TR bench.py --gpus 2 > gpurun_out/${T}_n2.json 2> gpurun_out/${T}_n2.err
timeout 600 $TR bench.py --gpus 2 --dims 2,1,1 --dtype f32 --no-e2e > gpurun_out/${T}_f32_n2_211.json 2> gpurun_out/${T}_f32_n2_211.err
timeout 600 $TR bench.py --gpus 2 --dims 2,1,1 --dtype f32 --fused-f32 --no-e2e > gpurun_out/${T}_f32f_n2_211.json 2> gpurun_out/${T}_f32f_n2_211.err
timeout 600 $TR bench.py --gpus 2 --workload acoustic --no-e2e > gpurun_out/${T}_ac_n2.json 2> gpurun_out/${T}_ac_n2.err
HALO_SIZES=${HALO_SIZES:-64,128,256,512,768} timeout 900 $TR scripts/halo_sweep.py > gpurun_out/${T}_halo.txt 2>&1
timeout 900 $TR scripts/b10_staggered.py > gpurun_out/${T}_b10.txt 2>&1
echo done
