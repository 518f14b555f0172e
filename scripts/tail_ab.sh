#!/bin/bash
# C5 at shard sizes of the strong split (1, 4, 8 GPUs) after routing non-simultaneous
# fallbacks straight to k_mc_small; parity subset of the lane/flat/fallback paths
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "c5 or c2 or lane or flat or zero or far or hint or worked or c1 or host or packed" > gpurun_out/tail_tests.log 2>&1; echo tests rc=$?; tail -n 1 gpurun_out/tail_tests.log
for ni in 1000000 250000 125000; do
    timeout 300 python bench.py --instances $ni --steps 10 --no-e2e --no-also --no-cpu-baseline > gpurun_out/tail_${ni}.json 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/tail_${ni}.json') if l.startswith('{')][-1])
print('n=$ni', '%.3g'%d['value'], round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"
done
timeout 300 python bench.py --workload c2 --steps 5 --no-e2e --no-also --no-cpu-baseline > gpurun_out/tail_c2.json 2>&1
python -c "
import json; d=json.loads([l for l in open('gpurun_out/tail_c2.json') if l.startswith('{')][-1])
print('c2', '%.3g'%d['value'], round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"
