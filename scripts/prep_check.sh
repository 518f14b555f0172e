#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -k "c3 or c4 or ring or invalid or hint or cap or worked or per_round or unmeasured or early or overestimate or packed or host or shard or zero or multirank" > gpurun_out/prep_tests.log 2>&1; echo tests_rc=$?; tail -n 2 gpurun_out/prep_tests.log
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_mcring.py > gpurun_out/san_prep_memcheck.txt 2>&1; echo memcheck rc=$?; tail -n 1 gpurun_out/san_prep_memcheck.txt
timeout 300 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_mcring.py > gpurun_out/san_prep_racecheck.txt 2>&1; echo racecheck rc=$?; tail -n 1 gpurun_out/san_prep_racecheck.txt
for wl in c4 c3; do for pol in mcsf mcbench; do
  timeout 400 python bench.py --workload $wl --policy $pol --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_${wl}_${pol}.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_${wl}_${pol}.json') if l.startswith('{')][-1])
print('$wl $pol', '%.3g'%d['value'], round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"
done; done
