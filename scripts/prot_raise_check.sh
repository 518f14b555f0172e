#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "protected or round2 or prot or early or overestimate" > gpurun_out/prot_tests.log 2>&1; echo tests_rc=$?; tail -n 2 gpurun_out/prot_tests.log
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python -c "
import sys; sys.path.insert(0,'.')
import workloads as W, paper_2502_07115_b200 as K
ctx=K.Context(0)
for eps in (0.2, 0.8):
    b=W.with_prediction_noise(W.c4(8, 5), eps, seed=3)
    g=K.simulate(ctx, b, K.Policy('mcsf_protected_raise', (1, 10)), hints=K.hints_of(b)); print(eps, g['status'])
" > gpurun_out/san_raise.txt 2>&1; echo san rc=$?; tail -n 3 gpurun_out/san_raise.txt
for pol in mcsf_protected mcsf_protected_raise; do for eps in 0.2 0.5 0.8; do
  timeout 600 python bench.py --workload c4 --policy $pol --eps $eps --steps 2 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_c4_${pol}_$eps.json 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_c4_${pol}_$eps.json') if l.startswith('{')][-1])
print('$pol $eps', '%.3g'%d['value'], round(d['ms_per_step'],2), 'ok', d['config']['instances_ok'], {k: round(v['ms_per_step'],2) for k,v in d['roofline']['kernels'].items()})"
done; done
