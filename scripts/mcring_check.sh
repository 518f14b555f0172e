#!/bin/bash
# GPU check of the 16-bit MC ring path: parity subset, C3/C4 bench lines (both MC policies)
# and the 32-bit k_ring A/B (KVSCHED_OLD_RING=1).  SAN=1 adds the sanitizers.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTS:-c3_trace or c4_large or ring or invalid or hint or cap or worked or per_round or unmeasured or early or overestimate or packed or host or shard or zero}" > gpurun_out/mcring_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/mcring_tests.log
if [ "$SAN" = 1 ]; then
for tool in memcheck racecheck synccheck; do
  timeout 300 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_mcring.py > gpurun_out/san_mcring_$tool.txt 2>&1; echo $tool rc=$?; tail -n 1 gpurun_out/san_mcring_$tool.txt
done
fi
for wl in c4 c3; do
  for pol in mcsf mcbench; do
    timeout 400 python bench.py --workload $wl --policy $pol --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_${wl}_${pol}.json 2>&1
  done
  [ "$AB" = 1 ] && KVSCHED_OLD_RING=1 timeout 400 python bench.py --workload $wl --steps 3 --no-e2e --no-also --no-cpu-baseline > gpurun_out/bench_${wl}_oldring.json 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_c[34]_*.json")):
    ls = [l for l in open(f) if l.startswith("{")]
    if not ls:
        print(f, "no line"); continue
    d = json.loads(ls[-1]); r = d["roofline"]
    print(f, "%.3g" % d["value"], round(d["ms_per_step"], 2), {k: round(v["ms_per_step"], 3) for k, v in r["kernels"].items()})
PY
