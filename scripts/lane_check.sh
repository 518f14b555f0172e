# GPU round trip for the lane kernel: build, parity subset, bench A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 240 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "c5 or c1 or c2 or fuzz or worked or per_round or invalid or maximum or shard or packed or host_path or lane or hint" > gpurun_out/pytest_lane.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_lane.log
timeout 240 python bench.py --ab --no-cpu-baseline --no-also --steps 10 > gpurun_out/bench_lane.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_lane.log
