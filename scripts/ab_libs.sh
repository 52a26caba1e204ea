# A/B of library builds on one GPU: LIBS="a b" (ablation/libigg_<x>.so; "cur" = the product library),
# bench.py arguments in ARGS, REPS runs each, interleaved -> gpurun_out/<TAG>_ab.txt
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; T=${TAG:-ab}
for rep in $(seq ${REPS:-3}); do
  for v in $LIBS; do
    L=ablation/libigg_$v.so; [ $v = cur ] && L=paper_2211_15716_b200/libigg.so
    r=$(IGG_LIBRARY=$L timeout 300 python bench.py $ARGS --no-e2e --no-cpu --no-stats 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round((d.get('exposed_halo') or {}).get('ms_per_step') or 0, 4))")
    echo "$v $ARGS: $r" >> gpurun_out/${T}_ab.txt
  done
done
