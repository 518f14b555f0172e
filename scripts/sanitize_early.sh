# compute-sanitizer memcheck / synccheck over the ring path's early-completion hand-off (k_ring -> k_prot)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "overestimate_ring and small" > gpurun_out/sanitizer_early_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_early_$tool.txt
done
