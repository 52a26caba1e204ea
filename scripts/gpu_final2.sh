cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/fn2_*
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fn2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/fn2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as G; G.smoke(); print('SMOKE OK')" > gpurun_out/fn2_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/fn2_n1.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fn2_ref.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2"
timeout 600 $R > gpurun_out/fn2_n2.log 2>&1
timeout 600 python bench.py --dtype f32 > gpurun_out/fn2_f32_n1.log 2>&1
for b in 16,2,2 0,0,0; do
  timeout 600 $R --dtype f32 --bw $b --no-e2e > gpurun_out/fn2_f32_n2_bw$b.log 2>&1
  echo "x-split bw$b $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/fn2_f32_n2_bw$b.log | head -1)" >> gpurun_out/fn2_f32.txt
done
timeout 600 $R --dtype f32 --no-e2e --fused-mode 8194 > gpurun_out/fn2_f32_n2_al.log 2>&1
echo "x-split aligned slabs $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/fn2_f32_n2_al.log | head -1)" >> gpurun_out/fn2_f32.txt
for d in 1,2,1 1,1,2; do
  timeout 600 $R --dtype f32 --no-e2e --dims $d > gpurun_out/fn2_f32_n2_d$d.log 2>&1
  echo "dims $d $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/fn2_f32_n2_d$d.log | head -1)" >> gpurun_out/fn2_f32.txt
done
echo done
