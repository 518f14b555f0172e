cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ring or c4 or c3 or alpha or long or fuzz or invalid or round_cap or host_path or protected" > gpurun_out/pytest_ring.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ring.log
for wl in "c4 mcsf" "c4 mcbench" "c4 alpha" "c4 alpha_beta" "c3 mcsf"; do set -- $wl
  timeout 600 python bench.py --workload $1 --policy $2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/br_$1_$2.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/br_$1_$2.log').read().strip().splitlines()[-1]); print('$1 $2', round(d['value']/1e9,3), round(d['ms_per_step'],2))"
done
