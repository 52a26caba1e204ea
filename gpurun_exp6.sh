cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp}
for cfg in "1,1,1:1,1,1" "1,2,1:0,0,0" "2,1,1:0,0,0"; do
  HT_DIMS=${cfg%%:*} HT_PER=${cfg#*:} timeout 300 python scripts/h26_trace.py >> gpurun_out/${T}_h26trace.txt 2>&1
done
echo done
