# ncu --set full of k_ring<MCSF> on a C4-shaped launch (2*10^4 instances)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ring -c 1 -o gpurun_out/prof_ring_c4 \
   python bench.py --workload c4 --instances 20000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-also > gpurun_out/ncu_ring.log 2>&1
echo "rc=$?"
timeout 300 python bench.py --workload c4 --instances 100000 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-also > gpurun_out/bench_c4.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_c4.log').read().strip().splitlines()[-1]); print(d['value']/1e9, d['ms_per_step'], d['roofline']['kernels'])"
