# acoustic_fused_kernel A/B (1 GPU): VARIANTS="cur ty2 ..." runs bench.py --workload acoustic twice per
# variant, cur = the product library, <v> = ablation/libigg_ac_<v>.so (built with
# python paper_2211_15716_b200/build.py --out ablation/libigg_ac_<v>.so -DIGG_ABLATION -DAF_TY=.. -DAF_KC=.. -DAF_D=..)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp}
for v in ${VARIANTS:-cur}; do
  L=ablation/libigg_ac_$v.so; [ $v = cur ] && L=paper_2211_15716_b200/libigg.so
  for rep in 1 2; do
  IGG_LIBRARY=$L timeout 300 python bench.py --workload acoustic --no-e2e --no-cpu --no-stats --steps 50 --warmup 5 > gpurun_out/${T}_$v.json 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_$v.json)" >> gpurun_out/${T}_summary.txt
  done
done
echo done
