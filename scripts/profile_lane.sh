# ncu --set full of the lane kernel (and its k_mc_small fallback launch) on the bench workload
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mc_ -s 2 -c 2 -o gpurun_out/prof_lane \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-also > gpurun_out/ncu_lane.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_lane.log
