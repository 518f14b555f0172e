cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "per_round or c5 or fuzz or worked or overestimate or large_queues or c1" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for mb in ${MBS:-8 10 12}; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DKV_SMALL_MIN_BLOCKS=$mb -I include -o /tmp/libkv_$mb.so paper_2502_07115_b200/csrc/kvsched.cu
  KVSCHED_LIB=/tmp/libkv_$mb.so timeout 600 python bench.py --steps 40 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_mb$mb.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_mb$mb.log').read().strip().splitlines()[-1]); print('mb=$mb', round(d['value']/1e9,2), round(d['ms_per_step'],3))"
done
