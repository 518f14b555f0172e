#!/bin/bash
# A/B of k_mc_ring build variants (KVSCHED_NVCC_DEFS) on C4 / C3, MC-SF and MC-Benchmark;
# parity subset on the default build first.  VARIANTS="name:-DX=1 name2:-DY=0"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTS:-c3_trace or c4_large or ring or worked or per_round or overestimate or cap or invalid or hint}" > gpurun_out/ring_tests.log 2>&1; echo tests_rc=$?; tail -n 1 gpurun_out/ring_tests.log
run() {
  for wl in ${WLS:-c4 c3}; do for pol in ${POLS:-mcsf}; do
    timeout 400 python bench.py --workload $wl --policy $pol --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ab_${1}_${wl}.json 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/ab_${1}_${wl}.json') if l.startswith('{')][-1])
print('$1 $wl $pol', '%.3g'%d['value'], round(d['ms_per_step'],2), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"
  done; done
}
run base
for v in $VARIANTS; do
  name=${v%%:*}; defs=${v#*:}
  KVSCHED_NVCC_DEFS="$defs" python -c "from paper_2502_07115_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  run $name
done
