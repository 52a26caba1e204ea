cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sched_*.log
B="python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --timeline"
timeout 300 $B > gpurun_out/sched_A_full.log 2>&1
timeout 300 $B --kernel 30 > gpurun_out/sched_A3_full_list.log 2>&1
timeout 300 $B --periodic 1,0,0 --bw 0,0,0 --skip-comm > gpurun_out/sched_B_seq_nocomm.log 2>&1
timeout 300 $B --periodic 1,0,0 --bw 2,2,2 --xalign 1 --skip-comm > gpurun_out/sched_D_split2_nocomm.log 2>&1
timeout 300 $B --periodic 1,0,0 --bw 16,2,2 --skip-comm > gpurun_out/sched_C_split64_nocomm.log 2>&1
timeout 300 $B --periodic 1,0,0 --bw 2,2,2 --xalign 1 > gpurun_out/sched_G_split2_selfwrap.log 2>&1
timeout 300 $B --periodic 1,1,1 --bw 2,2,2 --xalign 1 --skip-comm > gpurun_out/sched_H_split2_3ax_nocomm.log 2>&1
timeout 300 $B --periodic 1,1,1 --bw 16,2,2 > gpurun_out/sched_H2_split64_3ax.log 2>&1
echo done
