cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_default.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_check_split" -c 1 -o /tmp/split python bench.py --mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_ncu_split.log 2>&1
ncu -i /tmp/split.ncu-rep --page raw --csv > gpurun_out/split_raw.csv 2>&1
echo done
