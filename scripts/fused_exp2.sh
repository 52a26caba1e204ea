# 2-GPU fused-kernel experiment (gpurun --gpus 2): fused/virtual-rank GPU tests, 1-GPU periodic-x self-wrap
# bench, the three 2-GPU splits, a per-block trace of 2x1x1 (ablation/libigg_trace.so) and, with MULTI=1,
# the multi-GPU tests.  TAG names the outputs (gpurun_out/<TAG>_*).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-fx}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29525 --nproc-per-node 2"
timeout 600 python -m pytest tests -q -m gpu -x -k "virtual_p2p or fused or smoke" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python bench.py --periodic 1,0,0 --no-e2e --no-cpu --no-stats > gpurun_out/${T}_p100.json 2>&1
for d in 2,1,1 1,1,2 1,2,1; do
  timeout 600 $TR bench.py --gpus 2 --dims $d --no-e2e --no-stats > gpurun_out/${T}_n2_${d//,/}.json 2>&1
done
IGG_LIBRARY=ablation/libigg_trace.so timeout 300 $TR scripts/fused_trace2.py > gpurun_out/${T}_trace.txt 2>&1; mkdir -p gpurun_out/${T}_trace; mv gpurun_out/trace2_*.npz gpurun_out/${T}_trace/
TRACE_DIMS=1,2,1 IGG_LIBRARY=ablation/libigg_trace.so timeout 300 $TR scripts/fused_trace2.py > gpurun_out/${T}_trace_y.txt 2>&1; mkdir -p gpurun_out/${T}_trace_y; mv gpurun_out/trace2_*.npz gpurun_out/${T}_trace_y/
[ -n "$MULTI" ] && timeout 900 python -m pytest tests -q -m gpu -k "multi" > gpurun_out/${T}_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_multi.log
echo done
