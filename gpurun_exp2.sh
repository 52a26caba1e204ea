cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp12}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29525 --nproc-per-node 2"
timeout 600 python -m pytest tests -q -m gpu -x -k "acoustic_fused or acoustic_run" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python bench.py --workload acoustic --no-e2e --no-cpu --steps 20 > gpurun_out/${T}_ac.json 2>&1
timeout 300 python bench.py --no-e2e --no-cpu --no-stats > gpurun_out/${T}_n1.json 2>&1
timeout 600 $TR bench.py --gpus 2 --no-e2e --no-stats > gpurun_out/${T}_n2.json 2>&1
timeout 600 $TR bench.py --gpus 2 --no-e2e --no-stats --dims 1,2,1 > gpurun_out/${T}_n2_121.json 2>&1
echo done
