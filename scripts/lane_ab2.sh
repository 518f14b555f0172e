#!/bin/bash
# A/B of k_mc_lane build variants on the C5 bench (device path); lane parity subset first.
# VARIANTS="name:-DX=0 ..." (underscores in the defs become spaces)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTS:-lane or full_size_c5 or host_path_streamed}" > gpurun_out/lane_tests.log 2>&1; echo tests_rc=$?; tail -n 1 gpurun_out/lane_tests.log
run() {
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --no-also --no-cpu-baseline --no-e2e > gpurun_out/lab_$1.json 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/lab_$1.json') if l.startswith('{')][-1])
print('$1', '%.4g'%d['value'], round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"
  done
}
run base
for v in $VARIANTS; do
  name=${v%%:*}; defs=${v#*:}
  KVSCHED_NVCC_DEFS="${defs//_/ }" python -c "from paper_2502_07115_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  run $name
done
