#!/bin/bash
# Round-2 closing evidence after the CTA prep: smoke, full -m gpu suite, default bench line,
# reference arm, configs report, ncu of k_mc_ring on C3 (4096-slot window)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -n 1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 900 ncu --set full --import-source on -k regex:"k_mc_ring" -c 1 -o gpurun_out/ncu_final3_c3 python bench.py --workload c3 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 1800 python tests/tools/configs_report.py --out gpurun_out/configs_report.json > gpurun_out/configs_report.log 2>&1; echo "report rc=$?"
