# protected MC-SF (NEXT-1) on C4 + prediction noise: bench lines at three eps and an ncu capture of k_prot
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for eps in 0.2 0.5 0.8; do
  timeout 300 python bench.py --workload c4 --instances 20000 --policy mcsf_protected --eps $eps --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-also > gpurun_out/bench_prot_$eps.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_prot_$eps.log').read().strip().splitlines()[-1]); print('eps', $eps, d['value']/1e9, d['ms_per_step'], d['config']['instances_ok'], d['roofline']['kernel'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_prot -c 1 -o gpurun_out/prof_prot \
   python bench.py --workload c4 --instances 20000 --policy mcsf_protected --eps 0.2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-also > gpurun_out/ncu_prot.log 2>&1
echo "ncu rc=$?"
