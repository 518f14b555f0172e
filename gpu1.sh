set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q --maxfail=40 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench.log 2>&1
echo "bench rc=$?"
tail -3 gpurun_out/pytest_gpu.log
