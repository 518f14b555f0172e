cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on -k regex:k_mc_ring -c 1 -o gpurun_out/ncu_final_c3_mc_ring python bench.py --workload c3 --steps 1 --warmup 0 --no-e2e --no-also --no-cpu-baseline > gpurun_out/ncu_c3r.log 2>&1; echo "ncu c3 rc=$?"
KVSCHED_STREAM_TRACE=1 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 3 > gpurun_out/trace.json 2> gpurun_out/stream_trace.err; echo "trace rc=$?"
grep "stream trace" gpurun_out/stream_trace.err | tail -1 | cut -c1-200
