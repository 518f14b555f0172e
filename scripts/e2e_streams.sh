cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for ns in 2 3 4 6; do for rows in 2097152 4194304 8388608; do
  KVSCHED_HOST_STREAMS=$ns KVSCHED_HOST_CHUNK_ROWS=$rows timeout 300 python bench.py --no-cpu-baseline --no-also --steps 3 --e2e-steps 5 > gpurun_out/be.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/be.log').read().strip().splitlines()[-1]); print('streams', $ns, 'rows', $rows, round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_run'])"
done; done
