# One gpurun call of ncu captures (1 GPU; each command first runs plain and must exit 0):
#   launch list of the default bench, --set full of the production stencil (N=1), of the fused kernel
#   (periodic x+y+z self-wrap: every face kind), of the acoustic kernels, of the fused kernel with two
#   virtual 512^3 ranks (2x1x1: the cross-rank x data plane), and the 2R1W streaming probe.
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
VF="python scripts/virtual_fused.py"
timeout 300 $VF > gpurun_out/${T}_plain4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat_fused -s 3 -c 2 -o gpurun_out/${T}_prof_fused_virtual2 $VF > gpurun_out/${T}_ncu_fused_virtual2.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/stream_probe scripts/stream_probe.cu && timeout 300 /tmp/stream_probe > gpurun_out/${T}_stream_probe.txt 2>&1
timeout 300 python scripts/halo_local.py > gpurun_out/${T}_halo_local.txt 2>&1
HL_SIZES=64,512 HL_REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_halo_local_launches.csv python scripts/halo_local.py > gpurun_out/${T}_ncu_halo_local.log 2>&1
echo done
