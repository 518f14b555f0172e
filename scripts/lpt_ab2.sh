#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do
for w in 0 8 12 16; do
  KVSCHED_MCRING_WPS=$w timeout 400 python bench.py --workload c3 --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/lpt2_${w}.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/lpt2_${w}.json') if l.startswith('{')][-1])
print('c3 wps=$w', '%.3g'%d['value'], round(d['ms_per_step'],2), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()}, d['clocks'])"
done
done
KVSCHED_MCRING_WPS=12 timeout 400 python bench.py --workload c3 --policy mcbench --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/lpt2_b12.json 2>&1
KVSCHED_MCRING_WPS=0 timeout 400 python bench.py --workload c3 --policy mcbench --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/lpt2_b0.json 2>&1
for f in b12 b0; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/lpt2_$f.json') if l.startswith('{')][-1])
print('c3 mcbench $f', '%.3g'%d['value'], round(d['ms_per_step'],2))"; done
