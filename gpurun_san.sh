cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-san}
VARIANTS="cur ty2 ty8 ty8kc16 ty2kc64 kc64" TAG=${T}ac bash gpurun_exp4.sh
bash scripts/validate.sh $T san:memcheck san:racecheck san:synccheck
echo done
