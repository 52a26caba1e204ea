cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/sanitize_small.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python scripts/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/san_memcheck.log
echo done
