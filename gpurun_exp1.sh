cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp11}
timeout 900 python -m pytest tests -q -m gpu -x -k "virtual_p2p or fused or acoustic" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for per in 1,0,0 0,1,0 1,1,1; do
  echo "== $per" >> gpurun_out/${T}.txt
  timeout 300 python bench.py --periodic $per --no-e2e --no-cpu --no-stats --steps 100 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['exposed_halo'], d['roofline']['avg_launch_ms'])" >> gpurun_out/${T}.txt 2>&1
done
timeout 300 python bench.py --workload acoustic --no-e2e --no-cpu --steps 20 > gpurun_out/${T}_ac.json 2>&1
echo done
