#!/bin/bash
# GPU check of k_mc_flatq (C2): parity subset, sanitizers, C2 bench vs the one-lane k_mc_flat
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "c2 or lane or flat or c5 or zero or far or hint or worked or c1" > gpurun_out/flatq_tests.log 2>&1; echo tests_rc=$?; tail -n 3 gpurun_out/flatq_tests.log
if [ "$SAN" = 1 ]; then
for tool in memcheck racecheck synccheck; do
  timeout 300 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run3.py > gpurun_out/san_flatq_$tool.txt 2>&1; echo $tool rc=$?; tail -n 1 gpurun_out/san_flatq_$tool.txt
done
fi
for v in 0 1; do
  KVSCHED_FLAT_LANE=$v timeout 400 python bench.py --workload c2 --steps 5 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_c2_lane$v.json 2>&1
  KVSCHED_FLAT_LANE=$v timeout 400 python bench.py --workload c2 --policy mcbench --steps 5 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_c2b_lane$v.json 2>&1
  for f in bench_c2_lane$v bench_c2b_lane$v; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/$f.json') if l.startswith('{')][-1])
print('$f', '%.3g'%d['value'], round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"; done
done
