cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in "1,1,1:1,1,1" "1,2,1:0,0,0" "2,1,1:0,0,0"; do
  HT_DIMS=${cfg%%:*} HT_PER=${cfg#*:} timeout 300 python scripts/h26_trace.py >> gpurun_out/${T}_h26trace.txt 2>&1
done
for cfg in "1,1,1:1,1,1" "2,1,1:0,0,0" "2,1,1:1,1,1" "1,2,1:0,0,0" "2,2,2:0,0,0"; do
  d=${cfg%%:*}; p=${cfg#*:}
  echo "== dims $d per $p" >> gpurun_out/${T}_h26.txt
  HL_ONLY26=1 HL_DIMS=$d HL_PER=$p HL_SIZES=64,256,512 timeout 300 python scripts/halo_local.py >> gpurun_out/${T}_h26.txt 2>&1
done
echo done
