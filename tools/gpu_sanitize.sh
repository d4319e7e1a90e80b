# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py, both k_assign
# register variants (GAPLA_ASSIGN_VARIANT 0 / 1).  Logs in gpurun_out/sanitize_*.log.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 9"
for V in 0 1; do
  export GAPLA_ASSIGN_VARIANT=$V
  timeout 1500 $CS --tool memcheck --leak-check no python tools/sanitize_run.py > gpurun_out/sanitize_memcheck_v$V.log 2>&1
  echo "memcheck v$V rc=$?" >> gpurun_out/sanitize_summary.txt
  timeout 1500 $CS --tool synccheck python tools/sanitize_run.py cfg1_batch cfg1_flow bignets snapshot > gpurun_out/sanitize_synccheck_v$V.log 2>&1
  echo "synccheck v$V rc=$?" >> gpurun_out/sanitize_summary.txt
  timeout 2400 $CS --tool racecheck --racecheck-report all python tools/sanitize_run.py cfg1_batch cfg1_flow bignets snapshot > gpurun_out/sanitize_racecheck_v$V.log 2>&1
  echo "racecheck v$V rc=$?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
for f in gpurun_out/sanitize_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok \(|error|Error" $f | head -20; done
