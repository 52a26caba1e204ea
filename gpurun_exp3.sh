cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp}
timeout 900 python -m pytest tests -q -m gpu -x -k "acoustic" > gpurun_out/${T}_pytest_ac.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_ac.log
timeout 600 python bench.py --workload acoustic --no-e2e --no-cpu --no-stats > gpurun_out/${T}_ac.json 2>&1
HL_SIZES=64 HL_REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:halo26 -s 4 -c 1 -o gpurun_out/${T}_prof_h26 python scripts/halo_local.py > gpurun_out/${T}_ncu_h26.log 2>&1
echo done
