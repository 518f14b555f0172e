cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rows in 1048576 2097152 4194304 8388608 16777216; do
  KVSCHED_HOST_CHUNK_ROWS=$rows timeout 300 python bench.py --no-cpu-baseline --no-also --steps 3 --e2e-steps 5 > gpurun_out/bench_e2e.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_e2e.log').read().strip().splitlines()[-1]); print($rows, round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_run'])"
done
