cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_run3.py > gpurun_out/sanitize3_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "SUMMARY|done" gpurun_out/sanitize3_$tool.log
done
