cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for L in 256 512 1024 2048; do
  for wl in "c4 mcsf" "c4 mcbench" "c4 alpha_beta" "c3 mcsf"; do set -- $wl
    KVSCHED_RING_WINDOW=$L timeout 600 python bench.py --workload $1 --policy $2 --instances ${N:-0} --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bw_$L_$1_$2.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bw_$L_$1_$2.log').read().strip().splitlines()[-1]); print('L=$L $1 $2', round(d['value']/1e9,3), round(d['ms_per_step'],2))"
  done
done
