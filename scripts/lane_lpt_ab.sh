#!/bin/bash
# lane kernel: largest-first claim groups at strong-split shard sizes (+ DRAM bytes of the C5 launch)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "c5 or lane or worked or c1 or host or packed or hint or far" > gpurun_out/lanelpt_tests.log 2>&1; echo tests rc=$?; tail -n 1 gpurun_out/lanelpt_tests.log
for lpt in 0 1; do
for ni in 1000000 250000 125000; do
    KVSCHED_LANE_LPT=$lpt timeout 300 python bench.py --instances $ni --steps 10 --no-also --no-cpu-baseline --no-e2e > gpurun_out/lanelpt_${lpt}_${ni}.json 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/lanelpt_${lpt}_${ni}.json') if l.startswith('{')][-1])
print('lpt=$lpt n=$ni', '%.3g'%d['value'], round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['kernels'].items()})"
done; done
KVSCHED_LANE_LPT=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_mc_lane -s 1 -c 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-also > gpurun_out/lanelpt_dram.log 2>&1; grep -E "dram__bytes|gpu__time" gpurun_out/lanelpt_dram.log
