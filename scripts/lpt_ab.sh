#!/bin/bash
# A/B of longest-first claiming and resident warps per SM for k_mc_ring (C4, C3; MC-SF)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "c3_trace or c4_large or ring or worked or per_round or overestimate or cap or host" > gpurun_out/mcring_tests.log 2>&1; echo tests_rc=$?; tail -n 1 gpurun_out/mcring_tests.log
one() {   # label, env...
  local lab=$1; shift
  for wl in c4 c3; do
    env "$@" timeout 400 python bench.py --workload $wl --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/lpt_${lab}_${wl}.json 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/lpt_${lab}_${wl}.json') if l.startswith('{')][-1])
print('$lab $wl', '%.3g'%d['value'], round(d['ms_per_step'],2), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"
  done
}
one nolpt KVSCHED_LPT=0
one lpt_full KVSCHED_LPT=1
for w in 16 20 24 28; do one lpt_w$w KVSCHED_MCRING_WPS=$w; done
