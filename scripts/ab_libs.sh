# A/B two prebuilt library variants on the bench workload (experiments only)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_2502_07115_b200/lib
for v in "$@"; do
  cp $L/libkvsched_$v.so $L/libkvsched.so
  timeout 300 python bench.py --no-cpu-baseline --no-also --no-e2e --steps 10 > gpurun_out/bench_ab_$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_ab_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,1), round(d['ms_per_step'],3), {k: round(x['ms_per_step'],3) for k,x in d['roofline']['kernels'].items()})"
done
