# ncu --set full capture of C2's k_mc_flat launch (one GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mc_flat -s 1 -c 1 -o gpurun_out/prof_c2_flat \
   python bench.py --workload c2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-also > gpurun_out/ncu_c2.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/prof_c2_flat.ncu-rep --page details --csv > gpurun_out/prof_c2_flat_details.csv 2>&1
