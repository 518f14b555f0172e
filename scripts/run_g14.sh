# GPU round trip: build, smoke, gpu tests, optional extra command ($1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
# ncu evidence for the bench configuration (one GPU): launch list + full capture of the sim kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_mc_small -s 1 -c 1 -o gpurun_out/prof_bench_full \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ring -c 1 -o gpurun_out/prof_ring_c4 \
   python bench.py --workload c4 --instances 20000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ring.log 2>&1
echo "ring rc=$?"
timeout 900 python bench.py --steps 50 --warmup 5 --ab --e2e-steps 5 --cpu-seconds 10 > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
