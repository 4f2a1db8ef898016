cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 --records > gpurun_out/bench_c4_records.log 2>&1
echo done
