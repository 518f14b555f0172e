cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for L in 256 512 1024 2048; do
  KVSCHED_RING_WINDOW=$L timeout 600 python bench.py --workload c4 --policy mcsf_protected --eps 0.2 --instances 20000 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bp_$L.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bp_$L.log').read().strip().splitlines()[-1]); print('L=$L', round(d['value']/1e9,3), round(d['ms_per_step'],2))"
done
