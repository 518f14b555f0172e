cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mc_small -c 1 -o gpurun_out/prof_small \
   python bench.py --instances 100000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ls -la gpurun_out
