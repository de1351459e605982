# compute-sanitizer memcheck / racecheck / synccheck over the small-config cases of
# scripts/sanitize_case.py (every kernel path); logs to gpurun_out/${TAG}_san_<tool>.log
T=${TAG:-r02v}
export PYTORCH_NO_CUDA_MEMORY_CACHING=1  # torch frees at once: a leak report is then ours
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
timeout 900 $CS --tool memcheck --leak-check full python scripts/sanitize_case.py > gpurun_out/${T}_san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/${T}_san_memcheck.log
timeout 900 $CS --tool synccheck python scripts/sanitize_case.py > gpurun_out/${T}_san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/${T}_san_synccheck.log
timeout 1200 $CS --tool racecheck --racecheck-report analysis python scripts/sanitize_case.py c1 c1p ragged general cut both prof > gpurun_out/${T}_san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/${T}_san_racecheck.log
