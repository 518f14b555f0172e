#!/bin/bash
# Round-2 evidence: every config through the GPU path (configs report), ncu --set full of the
# new kernels (k_mc_ring on C4 and C3, k_mc_flatq on C2), the bench launch list + lane capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python tests/tools/configs_report.py --out gpurun_out/configs_report.json > gpurun_out/configs_report.log 2>&1; echo report rc=$?
timeout 600 ncu --set full --import-source on -k regex:k_mc_ring -c 1 -o gpurun_out/ncu_r02_c4_mc_ring python bench.py --workload c4 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo c4 rc=$?
timeout 900 ncu --set full --import-source on -k regex:k_mc_ring -c 1 -o gpurun_out/ncu_r02_c3_mc_ring python bench.py --workload c3 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo c3 rc=$?
timeout 600 ncu --set full --import-source on -k regex:k_mc_flatq -c 1 -o gpurun_out/ncu_r02_c2_flatq python bench.py --workload c2 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1; echo c2 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02.csv \
   python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-also > gpurun_out/bench_under_ncu.log 2>&1; echo launches rc=$?
