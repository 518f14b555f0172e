cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
