cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-exp}
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/stream_probe scripts/stream_probe.cu && timeout 300 /tmp/stream_probe > gpurun_out/${T}_stream_probe.txt 2>&1
for cfg in "1,1,1:1,1,1" "1,1,1:0,0,0" "2,1,1:0,0,0" "2,1,1:1,1,1" "1,2,1:0,0,0" "1,1,2:0,0,0" "2,2,2:0,0,0"; do
  d=${cfg%%:*}; p=${cfg#*:}
  echo "== dims $d per $p" >> gpurun_out/${T}_h26.txt
  HL_ONLY26=1 HL_DIMS=$d HL_PER=$p HL_SIZES=64,256 timeout 300 python scripts/halo_local.py >> gpurun_out/${T}_h26.txt 2>&1
done
VARIANTS="cur" bash gpurun_exp4.sh
echo done
