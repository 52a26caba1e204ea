cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp16}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29525 --nproc-per-node 2"
timeout 600 python -m pytest tests -q -m gpu -x -k "virtual_p2p or fused" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for lib in paper_2211_15716_b200/libigg.so ablation/libigg_scfence.so; do
  b=$(basename $lib .so)
  for d in 2,1,1 1,1,2; do
    IGG_LIBRARY=$lib timeout 600 $TR bench.py --gpus 2 --dims $d --no-e2e --no-stats > gpurun_out/${T}_${b}_n2_${d//,/}.json 2>&1
  done
done
echo done
