# One gpurun call of ncu captures (1 GPU; each command first runs plain and must exit 0):
#   launch list of the default bench, --set full of the production stencil (N=1), of the fused kernel
#   (periodic x+y+z self-wrap: every face kind), of the acoustic kernels and of the 26-neighbour update_halo.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; T=${TAG:-r02}
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-stats --no-exposed"
timeout 300 $B > gpurun_out/${T}_plain_launch.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 300 $B > gpurun_out/${T}_plain1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_box_async -s 3 -c 2 -o gpurun_out/${T}_prof_stencil $B > gpurun_out/${T}_ncu_stencil.log 2>&1
BF="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-stats --no-exposed --periodic 1,1,1"
timeout 300 $BF > gpurun_out/${T}_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_fused -s 3 -c 2 -o gpurun_out/${T}_prof_fused $BF > gpurun_out/${T}_ncu_fused.log 2>&1
BA="python bench.py --workload acoustic --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 300 $BA > gpurun_out/${T}_plain3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:acoustic -s 4 -c 2 -o gpurun_out/${T}_prof_acoustic $BA > gpurun_out/${T}_ncu_acoustic.log 2>&1
echo done
