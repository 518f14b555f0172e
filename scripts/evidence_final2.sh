#!/bin/bash
# Round-2 closing evidence after the CTA prep: smoke, full -m gpu suite, default bench line,
# reference arm, configs report, ncu of the C4 prep + ring
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -n 1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 600 ncu --set full --import-source on -k regex:"k_mc_prep|k_mc_ring" -c 3 -o gpurun_out/ncu_final2_c4 python bench.py --workload c4 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 1800 python tests/tools/configs_report.py --out gpurun_out/configs_report.json > gpurun_out/configs_report.log 2>&1; echo "report rc=$?"
