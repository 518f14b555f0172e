#!/bin/bash
# A/B of k_mc_ring build variants on C4 / C3 (MC-SF): KV_MCRING_MINB = 8 (64 regs) vs 10
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "c3_trace or c4_large or ring or worked or per_round or overestimate or cap" > gpurun_out/mcring_tests.log 2>&1; echo tests_rc=$?; tail -n 1 gpurun_out/mcring_tests.log
run() {
  for wl in c4 c3; do
    timeout 400 python bench.py --workload $wl --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ab_${1}_${wl}.json 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/ab_${1}_${wl}.json') if l.startswith('{')][-1])
print('$1 $wl', '%.3g'%d['value'], round(d['ms_per_step'],2), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"
  done
}
run base
for mb in ${MINBS:-10 12}; do
  KVSCHED_NVCC_DEFS="-DKV_MCRING_MINB=$mb" python -c "from paper_2502_07115_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  grep -A2 "k_mc_ringILi0" paper_2502_07115_b200/lib/ptxas.log | grep -E "registers|spill" | head -2
  run minb$mb
done
