# GPU round trip: build, smoke, gpu tests, optional extra command ($1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
grep -E "FAILED|Error|assert" gpurun_out/pytest_gpu.log | head -20
timeout 900 python bench.py --steps 30 --warmup 3 --e2e-steps 5 --cpu-seconds 8 > gpurun_out/bench_e2e.log 2>&1; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_e2e.log').read().strip().splitlines()[-1]); print(d['value']/1e9, d['ms_per_step'], d['e2e'])"
for eps in 0.2 0.5; do timeout 600 python bench.py --workload c4 --policy mcsf_protected --eps $eps --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_prot_$eps.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_prot_$eps.log').read().strip().splitlines()[-1]); print('prot eps $eps', d['value']/1e9, d['ms_per_step'], d['config']['instances_ok'])"; done
