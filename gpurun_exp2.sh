cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp13}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29525 --nproc-per-node 2"
IGG_LIBRARY=ablation/libigg_xdirect.so timeout 600 python -m pytest tests -q -m gpu -x -k "virtual_p2p or fused_self" > gpurun_out/${T}_pytest_xd.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_xd.log
for lib in paper_2211_15716_b200/libigg.so ablation/libigg_xdirect.so; do
  b=$(basename $lib .so)
  IGG_LIBRARY=$lib timeout 300 python bench.py --periodic 1,0,0 --no-e2e --no-cpu --no-stats > gpurun_out/${T}_${b}_p100.json 2>&1
  IGG_LIBRARY=$lib timeout 600 $TR bench.py --gpus 2 --no-e2e --no-stats > gpurun_out/${T}_${b}_n2.json 2>&1
  IGG_LIBRARY=$lib timeout 600 $TR bench.py --gpus 2 --no-e2e --no-stats > gpurun_out/${T}_${b}_n2b.json 2>&1
done
echo done
