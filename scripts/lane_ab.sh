# A/B: the in-tree library vs a previous build copied to ab/libkvsched_old.so (KVSCHED_LIB), C5 bench
# line, then the lane-kernel parity subset with the in-tree library
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/lane_ab.log
for i in 1 2 3; do
  for lib in old new; do
    if [ $lib = old ]; then export KVSCHED_LIB=$PWD/ab/libkvsched_old.so; else unset KVSCHED_LIB; fi
    timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-also \
      | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), '%.4e' % d['value'], d['roofline']['kernels'].get('k_mc_lane<MCSF>'))" >> gpurun_out/lane_ab.log 2>&1
  done
done
unset KVSCHED_LIB
cat gpurun_out/lane_ab.log
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "lane or scope or c5 or C5 or packed or host" > gpurun_out/lane_tests.log 2>&1
tail -1 gpurun_out/lane_tests.log
