# e2e sweep: grid share, compute streams, chunk rows (experiments)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "4 4 4194304" "1 2 12582912" "2 2 12582912" "1 4 12582912" "2 4 8388608" "1 2 25165824" "3 3 6291456"; do
  set -- $cfg
  KVSCHED_HOST_GRID_DIV=$1 KVSCHED_HOST_STREAMS=$2 KVSCHED_HOST_CHUNK_ROWS=$3 timeout 300 python bench.py --no-cpu-baseline --no-also --steps 3 --e2e-steps 5 > gpurun_out/be.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/be.log').read().strip().splitlines()[-1]); print('div', $1, 'streams', $2, 'rows', $3, round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_run'])"
done
