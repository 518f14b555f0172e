# A/B: k_mc_flat launch shape (ab/libkvsched_old.so = previous build via KVSCHED_LIB) on C2 and C5,
# then the flat/C2 parity subset with the in-tree library
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
rm -f gpurun_out/flat_ab.log
for i in 1 2 3; do
  for lib in old new; do
    if [ $lib = old ]; then export KVSCHED_LIB=$PWD/ab/libkvsched_old.so; else unset KVSCHED_LIB; fi
    for wl in c2 c5; do
      timeout 300 python bench.py --workload $wl --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-also \
        | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib $wl', round(d['ms_per_step'],4), '%.4e' % d['value'], d['roofline']['kernels'])" >> gpurun_out/flat_ab.log 2>&1
    done
  done
done
unset KVSCHED_LIB
cat gpurun_out/flat_ab.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "flat or c2 or C2 or scope or c5 or C5" > gpurun_out/flat_tests.log 2>&1
tail -1 gpurun_out/flat_tests.log
