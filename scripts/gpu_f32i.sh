cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/h38_*
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dtype f32 --steps 100 --warmup 10 --no-e2e"
for cfg in "--bw 2,2,2 --fused-mode 16386" "--bw 4,2,2 --fused-mode 16386" "--bw 16,2,2" "--bw 2,2,2 --fused-mode 16386" "--bw 2,2,2 --fused-mode 16386 --dims 1,2,1"; do
  tag=$(echo $cfg | tr -d ' -' | tr ',' '_')
  timeout 600 $R $cfg > gpurun_out/h38_$tag.log 2>&1
  echo "$cfg $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/h38_$tag.log | head -1) $(grep -o '"exposed_halo": {[^}]*}' gpurun_out/h38_$tag.log)" >> gpurun_out/h38_sum.txt
done
echo done
