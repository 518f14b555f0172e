# GPU round trip: build, smoke, gpu tests, optional extra command ($1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head; timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; python -c "import json; d=json.loads(open(\"gpurun_out/bench_default.log\").read().strip().splitlines()[-1]); print(d[\"value\"]/1e9, d[\"e2e\"])"
