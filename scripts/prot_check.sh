# protected MC-SF: parity tests + bench (jump vs per-round)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "protected or prot" -p no:cacheprovider > gpurun_out/pytest_prot.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_prot.log
for f in 0 1; do
  timeout 600 python bench.py --workload c4 --policy mcsf_protected --eps 0.2 --instances 20000 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline $( [ $f = 1 ] && echo --ab ) > gpurun_out/bp_f$f.log 2>&1
  tail -1 gpurun_out/bp_f$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('f=$f', d['value'], d['ms_per_step'], d.get('ab'))"
done
