#!/bin/bash
# GPU check of the 16-bit MC ring path: parity subset, sanitizers, C3/C4 bench lines and A/B
# against the 32-bit k_ring (KVSCHED_OLD_RING=1).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "c3 or c4 or ring or invalid or hint or cap or worked or per_round or unmeasured or early or overestimate or packed or host or shard or zero" > gpurun_out/mcring_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/mcring_tests.log
for tool in memcheck racecheck synccheck; do
  timeout 300 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_mcring.py > gpurun_out/san_mcring_$tool.txt 2>&1; echo $tool rc=$?; tail -2 gpurun_out/san_mcring_$tool.txt
done
for wl in c4 c3; do
  timeout 400 python bench.py --workload $wl --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_${wl}_mcring.json 2>&1
  KVSCHED_OLD_RING=1 timeout 400 python bench.py --workload $wl --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_${wl}_oldring.json 2>&1
  timeout 400 python bench.py --workload $wl --policy mcbench --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_${wl}_mcring_bench.json 2>&1
done
