#!/bin/bash
# streamed host path: parity through the host entry point (all formats, chunk counts), a
# sanitizer pass, then the bench's e2e (streamed vs the chunked pipeline)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k "host or packed" > gpurun_out/stream_tests.log 2>&1; echo tests rc=$?; tail -n 2 gpurun_out/stream_tests.log
KVSCHED_HOST_STREAM_CHUNKS=5 timeout 600 python -m pytest tests -m gpu -x -q -k "host or packed" > gpurun_out/stream_tests5.log 2>&1; echo tests5 rc=$?; tail -n 1 gpurun_out/stream_tests5.log
timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python scripts/sanitize_run3.py > gpurun_out/san_stream.txt 2>&1; echo san rc=$?; tail -n 2 gpurun_out/san_stream.txt
for v in 1 0; do for rep in 1 2; do
  KVSCHED_HOST_STREAM=$v timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/stream_e2e.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/stream_e2e.json') if l.startswith('{')][-1])
print('stream=$v', 'device ms', round(d['ms_per_step'],3), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'match', d['e2e']['matches_device_run'])" || tail -5 gpurun_out/stream_e2e.json
done; done
