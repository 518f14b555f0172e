#!/bin/bash
# Round-2 final evidence: smoke, the full -m gpu suite, the default bench line, every config
# (configs report), ncu --set full of the bench kernel and of k_mc_ring / k_mc_prep (C4, C3),
# the bench launch list, a randomized parity sweep (incl. the streamed host path)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -n 1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2>&1; echo "ref rc=$?"
# (compute-sanitizer is closed on this GPU pool; the streamed path's parity is covered by the
# tests and the randomized sweep below)
timeout 900 python tests/tools/fuzz_parity.py 8 > gpurun_out/fuzz_stdout.log 2>&1; echo "fuzz rc=$?"; tail -n 1 gpurun_out/fuzz_parity.log
timeout 600 ncu --set full --import-source on -k regex:k_mc_lane -c 1 -o gpurun_out/ncu_final_bench_lane python bench.py --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_lane.log 2>&1; echo "ncu lane rc=$?"
timeout 600 ncu --set full --import-source on -k regex:k_mc_ring -c 1 -o gpurun_out/ncu_final_c4_mc_ring python bench.py --workload c4 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --import-source on -k regex:"k_mc_ring|k_mc_prep" -c 2 -o gpurun_out/ncu_final_c3 python bench.py --workload c3 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_final.csv \
   python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-also > gpurun_out/bench_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 1800 python tests/tools/configs_report.py --out gpurun_out/configs_report.json > gpurun_out/configs_report.log 2>&1; echo "report rc=$?"; tail -n 3 gpurun_out/configs_report.log
