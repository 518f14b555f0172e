# GPU round trip: build, smoke, gpu tests, optional extra command ($1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head -20
for wl in "c4 mcsf" "c4 mcbench" "c4 alpha" "c4 alpha_beta" "c3 mcsf"; do set -- $wl
  timeout 600 python bench.py --workload $1 --policy $2 --steps 5 --warmup 2 --ab --no-e2e --no-cpu-baseline > gpurun_out/bench_$1_$2.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_$1_$2.log').read().strip().splitlines()[-1]); print('$1 $2', round(d['value']/1e9,3), 'G rounds/s', round(d['ms_per_step'],2), 'ms', d['roofline']['kernel'], 'ab', d['ab'] and round(d['ab']['speedup_of_default'],2))" 2>&1 | tail -1
done
