# GPU round trip: build, smoke, gpu tests, optional extra command ($1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head; timeout 1200 python tools/configs_report.py --out gpurun_out/configs_report.json > gpurun_out/configs_report.log 2>&1; echo "report rc=$?"; grep C2 gpurun_out/configs_report.log | cut -c1-700
