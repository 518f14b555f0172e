cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q --maxfail=40 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 50 --warmup 5 --ab --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/pytest_gpu.log
