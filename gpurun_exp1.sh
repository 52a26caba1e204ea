cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp10}
for lib in paper_2211_15716_b200/libigg.so ablation/libigg_natural.so; do
for per in 1,0,0 0,1,0 0,0,1 1,1,1; do
  echo "== $lib $per" >> gpurun_out/${T}.txt
  IGG_LIBRARY=$lib timeout 300 python bench.py --periodic $per --no-e2e --no-cpu --no-stats --steps 100 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['exposed_halo'], d['roofline']['avg_launch_ms'])" >> gpurun_out/${T}.txt 2>&1
done; done
for v in trace trace_natural; do
  IGG_LIBRARY=ablation/libigg_${v}.so timeout 600 python scripts/fused_trace.py > gpurun_out/${T}_${v}.txt 2>&1; mkdir -p gpurun_out/${T}_${v}; mv gpurun_out/trace_*.npz gpurun_out/${T}_${v}/
done
echo done
