cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ring -c 1 -o gpurun_out/prof_ring_c3 \
   python bench.py --workload c3 --instances 512 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
echo "rc=$?"
