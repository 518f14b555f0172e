# ncu source-level profile of k_mc_small using the shipped (locally built) library
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mc_small -c 1 -o gpurun_out/prof_small_src \
   python bench.py --instances 100000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_src.log 2>&1
echo "rc=$?"
