cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp14}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29525 --nproc-per-node 2"
for v in trace trace_xd; do
  IGG_LIBRARY=ablation/libigg_${v}.so timeout 300 $TR scripts/fused_trace2.py > gpurun_out/${T}_${v}.txt 2>&1; mkdir -p gpurun_out/${T}_${v}; mv gpurun_out/trace2_*.npz gpurun_out/${T}_${v}/
done
timeout 600 python -m pytest tests -q -m gpu -x -k "acoustic" > gpurun_out/${T}_pytest_ac.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_ac.log
timeout 300 python bench.py --workload acoustic --no-e2e --no-cpu --steps 20 > gpurun_out/${T}_ac.json 2>&1
echo done
