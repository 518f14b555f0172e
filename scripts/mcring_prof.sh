#!/bin/bash
# ncu --set full of k_mc_ring (C4, C3) and the per-line table of the C4 capture
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on -k regex:k_mc_ring -c 1 -o gpurun_out/ncu_c4_mcring python bench.py --workload c4 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c4_mcring.log 2>&1; echo ncu_c4=$?
[ "$C3" = 1 ] && timeout 900 ncu --set full --import-source on -k regex:k_mc_ring -c 1 -o gpurun_out/ncu_c3_mcring python bench.py --workload c3 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c3_mcring.log 2>&1; echo ncu_c3=$?
