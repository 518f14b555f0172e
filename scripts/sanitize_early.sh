# compute-sanitizer memcheck / racecheck / synccheck over the ring path: the early-completion
# hand-off (k_ring -> k_prot), k_ring<MCSF> with the next-head prefetch, and k_prot
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
SEL="(overestimate_ring and small) or (c4_policies and mcsf) or (protected_mcsf and small and 0.2)"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$SEL" > gpurun_out/sanitizer_ring_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_ring_$tool.txt
done
