#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on -k regex:k_mc_prep -c 2 -o gpurun_out/ncu_c4_prep python bench.py --workload c4 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c4_prep.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --import-source on -k regex:k_mc_prep -c 2 -o gpurun_out/ncu_c3_prep python bench.py --workload c3 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c3_prep.log 2>&1; echo ncu=$?
