# GPU round trip: build + smoke, full -m gpu suite, default bench line (C5 + C2/C4/C3 beside it)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 2 gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q --maxfail=10 -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -n 2
[ "$PROFILE" = 1 ] && bash scripts/profile_bench.sh
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l = [x for x in open("gpurun_out/bench_default.log") if x.startswith("{")]
d = json.loads(l[-1])
print("C5", "%.3g" % d["value"], round(d["ms_per_step"], 3), "e2e %.3g" % d["e2e"]["value"], "frac", round(d["roofline"]["frac"], 3))
for k, v in (d.get("other_configs") or {}).items():
    print(k, "%.3g" % v["value"], round(v["ms_per_step"], 3), v["kernels_ms_per_step"])
print("cpu", d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"], d["clocks"])
PY
