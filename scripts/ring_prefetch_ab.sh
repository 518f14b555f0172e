# A/B: k_ring head-entry prefetch (new, in-tree build) vs the previous library (ab/libkvsched_old.so), C4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ring_ab.log
for i in 1 2; do
  for pol in mcsf_protected; do
    for lib in old new; do
      if [ $lib = old ]; then export KVSCHED_LIB=$PWD/ab/libkvsched_old.so; else unset KVSCHED_LIB; fi
      timeout 300 python bench.py --workload c4 --instances 20000 --policy $pol --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-also \
        | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$pol $lib', round(d['ms_per_step'],3), '%.3e' % d['value'])" >> gpurun_out/ring_ab.log 2>&1
    done
  done
done
unset KVSCHED_LIB
cat gpurun_out/ring_ab.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "protected or overestimate or maximum" > gpurun_out/ring_tests.log 2>&1
tail -1 gpurun_out/ring_tests.log
