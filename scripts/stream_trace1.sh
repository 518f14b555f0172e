cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
KVSCHED_STREAM_TRACE=1 timeout 300 python bench.py --steps 3 --no-also --no-cpu-baseline --e2e-steps 3 > gpurun_out/trace.json 2> gpurun_out/trace.err
grep "stream trace" gpurun_out/trace.err | tail -1
