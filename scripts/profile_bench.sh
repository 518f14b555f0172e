# ncu evidence for the bench configuration (one GPU): launch list + full capture of the
# simulation kernels of one timed step (k_mc_lane, k_mc_flat and the k_mc_small fallback launches)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-also > gpurun_out/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mc_ -s 4 -c 4 -o gpurun_out/prof_bench_lane \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-also > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
