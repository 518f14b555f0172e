# GPU round trip: build + smoke, full -m gpu suite, default bench line, ncu evidence of the bench launch
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q --maxfail=10 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
bash scripts/profile_bench.sh          # ncu first: bench.py reads the capture for its roofline
timeout 400 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 400 python bench.py --ab --no-cpu-baseline --no-e2e --no-also > gpurun_out/bench_ab.log 2>&1; echo "ab rc=$?"

