cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "ring or c4 or c3 or long or fuzz or very_ragged or maximum or worked" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_sel.log
for pol in mcsf mcbench; do
  timeout 300 python bench.py --workload c4 --instances 100000 --policy $pol --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-also > gpurun_out/bc4.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bc4.log').read().strip().splitlines()[-1]); print('c4', '$pol', d['value']/1e9, d['ms_per_step'])"
done
