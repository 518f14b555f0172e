#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on -k regex:k_mc_flat -c 1 -o gpurun_out/ncu_c2_flatq python bench.py --workload c2 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c2_flatq.log 2>&1; echo ncu=$?
