#!/bin/bash
# host-path pipeline sweep: compute streams x grid share x chunk rows x lane claim order
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
run() {  # streams griddiv chunkrows lpt
  KVSCHED_HOST_STREAMS=$1 KVSCHED_HOST_GRID_DIV=$2 KVSCHED_HOST_CHUNK_ROWS=$3 KVSCHED_LANE_LPT=$4 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/e2es.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/e2es.json') if l.startswith('{')][-1])
print('streams=$1 div=$2 rows=$3 lpt=$4', 'e2e ms', round(d['e2e']['ms_per_step'],3))"
}
run 4 4 4194304 0
run 4 4 4194304 1
run 2 1 8388608 1
run 2 2 8388608 1
run 3 1 6291456 1
run 4 2 4194304 1
run 2 1 12582912 1
run 6 2 2097152 1
run 4 4 2097152 0
