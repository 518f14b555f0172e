#!/bin/bash
# C2 A/B: k_mc_flat (one lane per instance) vs k_mc_flatq with 4 / 8 / 16 lanes per instance
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in 8 4 2; do
  KVSCHED_FLAT_LANE=$v timeout 900 python -m pytest tests -m gpu -x -q -k "c2 or flat or lane_scope or zero" > gpurun_out/flatq_tests_$v.log 2>&1; echo "tests G-code $v rc=$?"; tail -n 1 gpurun_out/flatq_tests_$v.log
done
for v in 1 4 8 2; do
  KVSCHED_FLAT_LANE=$v timeout 400 python bench.py --workload c2 --steps 5 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_c2_v$v.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_c2_v$v.json') if l.startswith('{')][-1])
print('C2 v$v', '%.3g'%d['value'], round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"
done
