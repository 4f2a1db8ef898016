cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_s2 -c 1 -o /tmp/s2_full python bench.py --suite 2 --log2n 24 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_ncu_s2.log 2>&1
ncu -i /tmp/s2_full.ncu-rep --page raw --csv > gpurun_out/s2_full_raw.csv 2>&1
ncu -i /tmp/s2_full.ncu-rep --page source --csv > gpurun_out/s2_full_source.csv 2>&1
echo done
