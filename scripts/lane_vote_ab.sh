# A/B: k_mc_lane profile shift with (ab/libkvsched_b32.so) and without (ab/libkvsched_w8.so, -DKV_LANE_SHIFT_VOTE=0)
# the warp-uniform stage skip, on C5; then the lane parity subset on the no-vote build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
rm -f gpurun_out/lane_vote_ab.log
for i in 1 2; do
  for lib in b32 w8 b32 w8; do
    if [ $lib = new ]; then unset KVSCHED_LIB; else export KVSCHED_LIB=$PWD/ab/libkvsched_$lib.so; fi
    timeout 300 python bench.py --workload c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-also \
      | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib c2', round(d['ms_per_step'],4), '%.4e' % d['value'], d['roofline']['kernels'].get('k_mc_lane<MCSF>'))" >> gpurun_out/lane_vote_ab.log 2>&1
  done
done
unset KVSCHED_LIB
cat gpurun_out/lane_vote_ab.log
for lib in w8; do
  if [ $lib = new ]; then unset KVSCHED_LIB; else export KVSCHED_LIB=$PWD/ab/libkvsched_$lib.so; fi
  timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "lane or scope or c5 or C5 or packed" > gpurun_out/lane_vote_tests_$lib.log 2>&1
  echo $lib; tail -1 gpurun_out/lane_vote_tests_$lib.log
done
