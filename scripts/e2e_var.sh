#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 5 --no-also --no-cpu-baseline --e2e-steps 5 > gpurun_out/e2e_$rep.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/e2e_$rep.json') if l.startswith('{')][-1])
print('rep $rep default', round(d['ms_per_step'],3), 'e2e ms', round(d['e2e']['ms_per_step'],3))"
done
