#!/bin/bash
# streamed host path: event timeline (KVSCHED_STREAM_TRACE) and e2e over chunk counts / SM reserve
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
KVSCHED_STREAM_TRACE=1 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 3 > gpurun_out/trace.json 2> gpurun_out/trace.err
grep "stream trace" gpurun_out/trace.err | tail -1
for cfg in "16 8 96 1" "12 8 96 1" "20 8 96 1" "16 10 96 1" "16 8 96 2"; do
  set -- $cfg
  KVSCHED_HOST_STREAM_CHUNKS=$1 KVSCHED_STREAM_RESERVE=$2 KVSCHED_STREAM_SIDE_BLOCKS=$3 KVSCHED_HOST_STREAM_GROUP=$4 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/sw.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/sw.json') if l.startswith('{')][-1])
print('chunks $1 reserve $2 side $3 group $4', 'e2e ms', round(d['e2e']['ms_per_step'],3), 'match', d['e2e']['matches_device_run'])" || tail -5 gpurun_out/sw.json
done
KVSCHED_HOST_STREAM=0 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/sw0.json 2>&1; python -c "
import json; d=json.loads([l for l in open(\"gpurun_out/sw0.json\") if l.startswith(\"{\")][-1]); print(\"chunked e2e ms\", round(d[\"e2e\"][\"ms_per_step\"],3))"
