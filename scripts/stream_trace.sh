#!/bin/bash
# streamed host path: event timeline (KVSCHED_STREAM_TRACE) and e2e over flag chunks / group size
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
KVSCHED_HOST_STREAM_CHUNKS=64 KVSCHED_HOST_STREAM_GROUP=4 KVSCHED_STREAM_TRACE=1 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 3 > gpurun_out/trace.json 2> gpurun_out/trace.err
grep "stream trace" gpurun_out/trace.err | tail -1
for cfg in "16 1" "64 4" "32 2" "128 8" "48 3"; do
  set -- $cfg
  KVSCHED_HOST_STREAM_CHUNKS=$1 KVSCHED_HOST_STREAM_GROUP=$2 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/sw.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/sw.json') if l.startswith('{')][-1])
print('chunks $1 group $2', 'e2e ms', round(d['e2e']['ms_per_step'],3), 'match', d['e2e']['matches_device_run'])" || tail -5 gpurun_out/sw.json
done
