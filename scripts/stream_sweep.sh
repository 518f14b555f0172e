#!/bin/bash
# streamed host path: parity (host/packed tests), then e2e over the SM reserve / side-grid split
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "host or packed" > gpurun_out/stream_tests.log 2>&1; echo tests rc=$?; tail -n 3 gpurun_out/stream_tests.log
for cfg in ${CFGS:-"6 24" "8 32" "12 48" "12 96" "20 160"}; do
  set -- $cfg
  KVSCHED_STREAM_RESERVE=$1 KVSCHED_STREAM_SIDE_BLOCKS=$2 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/sw.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/sw.json') if l.startswith('{')][-1])
print('reserve $1 side $2', 'e2e ms', round(d['e2e']['ms_per_step'],3), 'match', d['e2e']['matches_device_run'])" || tail -5 gpurun_out/sw.json
done
KVSCHED_HOST_STREAM=0 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/sw0.json 2>&1
python -c "
import json; d=json.loads([l for l in open('gpurun_out/sw0.json') if l.startswith('{')][-1])
print('chunked e2e ms', round(d['e2e']['ms_per_step'],3))"
