# GPU round trip: the default bench line (as the driver runs it) and the A/B variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 400 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 400 python bench.py --ab --no-cpu-baseline --no-e2e --no-also > gpurun_out/bench_ab.log 2>&1; echo "ab rc=$?"
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -c 400 gpurun_out/bench_default.log
