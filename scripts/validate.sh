#!/bin/bash
# One parametrised GPU validation script (run under gpurun from the repo root):
#   scripts/validate.sh <tag> <step>...      steps, run in order, each under its own timeout:
#     tests        pytest -m gpu                            -> gpurun_out/<tag>_pytest_gpu.log
#     tests:<k>    pytest -m gpu -k <k>                     -> gpurun_out/<tag>_pytest_<k>.log
#     smoke        __graft_entry__.smoke()                  -> gpurun_out/<tag>_smoke.log
#     bench        bench.py (N=1 defaults)                  -> gpurun_out/<tag>_n1.json
#     ref          bench.py --impl reference                -> gpurun_out/<tag>_ref.json
#     bench2/4     torchrun bench.py --gpus 2/4             -> gpurun_out/<tag>_n2.json / _n4.json
#     acoustic     bench.py --workload acoustic             -> gpurun_out/<tag>_ac_n1.json
#     f32          bench.py --dtype f32                     -> gpurun_out/<tag>_f32_n1.json
#     launches     plain bench, then ncu launch list        -> gpurun_out/<tag>_launches.csv
#     ncu:<regex>  plain bench, then ncu --set full of the first 3 matching launches -> <tag>_prof.ncu-rep
#     halo2/4      update_halo sweep (scripts/halo_sweep.py) -> gpurun_out/<tag>_halo_n2.txt
#     san:<tool>   compute-sanitizer --tool <tool> (memcheck | racecheck | synccheck; ONE per call) of
#                  scripts/sanitize_small.py, after a plain run of it -> gpurun_out/<tag>_san_<tool>.log
# Extra bench.py arguments: BENCH_ARGS="..." (plain runs and the ncu runs).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=$1; shift
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29517"
for step in "$@"; do
  case $step in
    tests) timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${tag}_pytest_gpu.log 2>&1
           echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log ;;
    tests:*) k=${step#tests:}; timeout 900 python -m pytest tests -q -m gpu -k "$k" > gpurun_out/${tag}_pytest_${k//[^a-zA-Z0-9_]/_}.log 2>&1
           echo "rc=$?" >> gpurun_out/${tag}_pytest_${k//[^a-zA-Z0-9_]/_}.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as G; G.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
           echo "rc=$?" >> gpurun_out/${tag}_smoke.log ;;
    bench) timeout 600 python bench.py $BENCH_ARGS > gpurun_out/${tag}_n1.json 2> gpurun_out/${tag}_n1.err ;;
    ref) timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err ;;
    bench2) timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 $BENCH_ARGS > gpurun_out/${tag}_n2.json 2> gpurun_out/${tag}_n2.err ;;
    bench4) timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 $BENCH_ARGS > gpurun_out/${tag}_n4.json 2> gpurun_out/${tag}_n4.err ;;
    acoustic) timeout 600 python bench.py --workload acoustic $BENCH_ARGS > gpurun_out/${tag}_ac_n1.json 2> gpurun_out/${tag}_ac_n1.err ;;
    f32) timeout 600 python bench.py --dtype f32 $BENCH_ARGS > gpurun_out/${tag}_f32_n1.json 2> gpurun_out/${tag}_f32_n1.err ;;
    launches) B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-stats $BENCH_ARGS"
           timeout 300 $B > gpurun_out/${tag}_plain.log 2>&1 && \
           timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
             --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/${tag}_ncu_launch.log 2>&1 ;;
    ncu:*) k=${step#ncu:}; B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-stats --no-exposed $BENCH_ARGS"
           timeout 300 $B > gpurun_out/${tag}_plain_full.log 2>&1 && \
           timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 3 \
             -o gpurun_out/${tag}_prof $B > gpurun_out/${tag}_ncu_full.log 2>&1 ;;
    halo2) timeout 600 $TR --nproc-per-node 2 scripts/halo_sweep.py > gpurun_out/${tag}_halo_n2.txt 2>&1 ;;
    halo4) timeout 600 $TR --nproc-per-node 4 scripts/halo_sweep.py > gpurun_out/${tag}_halo_n4.txt 2>&1 ;;
    san:*) tool=${step#san:}
           timeout 300 python scripts/sanitize_small.py > gpurun_out/${tag}_san_plain.log 2>&1 && \
           timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_small.py \
             > gpurun_out/${tag}_san_${tool}.log 2>&1
           echo "rc=$?" >> gpurun_out/${tag}_san_${tool}.log ;;
    *) echo "unknown step $step" ;;
  esac
done
echo "validate $tag done"
