#!/bin/bash
# streamed host path: parity through the host entry point (formats, chunk counts), then the
# bench's e2e, streamed (default) vs the chunked pipeline (KVSCHED_HOST_STREAM=0)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "host or packed" > gpurun_out/stream_tests.log 2>&1; echo tests rc=$?; tail -n 3 gpurun_out/stream_tests.log
for v in 1 0 1; do
  KVSCHED_HOST_STREAM=$v timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/stream_e2e_$v.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/stream_e2e_$v.json') if l.startswith('{')][-1])
print('stream=$v', 'device ms', round(d['ms_per_step'],3), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'match', d['e2e']['matches_device_run'])" || tail -5 gpurun_out/stream_e2e_$v.json
done
