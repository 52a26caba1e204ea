# A/B of library builds on 2 GPUs (gpurun --gpus 2): LIBS="a b" (ablation/libigg_<x>.so; "cur" = product),
# bench.py arguments in ARGS, REPS interleaved runs -> gpurun_out/<TAG>_ab2.txt
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; T=${TAG:-ab}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29541 --nproc-per-node 2"
for rep in $(seq ${REPS:-2}); do
  for v in $LIBS; do
    L=ablation/libigg_$v.so; [ $v = cur ] && L=paper_2211_15716_b200/libigg.so
    r=$(IGG_LIBRARY=$L timeout 300 $TR bench.py --gpus 2 $ARGS --no-e2e --no-cpu --no-stats 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round((d.get('exposed_halo') or {}).get('ms_per_step') or 0, 4))")
    echo "$v $ARGS: $r" >> gpurun_out/${T}_ab2.txt
  done
done
