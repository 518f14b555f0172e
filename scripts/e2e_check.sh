# GPU round trip: host-path parity tests + the bench e2e number
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python -m pytest tests -m gpu -q --maxfail=5 -p no:cacheprovider -k "host or packed or latency" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_sel.log
for rows in 0 2097152 8388608; do
  KVSCHED_HOST_CHUNK_ROWS=$rows timeout 300 python bench.py --no-cpu-baseline --no-also --steps 5 > gpurun_out/bench_e2e_$rows.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_e2e_$rows.log').read().strip().splitlines()[-1]); print($rows, d['value']/1e9, d['e2e']['ms_per_step'], d['e2e']['matches_device_run'])"
done
