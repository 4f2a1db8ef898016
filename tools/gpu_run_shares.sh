cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py --varlen --mode epoch --n2 1024 --log2n 25 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4_share.log 2>&1
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 27 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_share.log 2>&1
timeout 900 python bench.py --mode tamper --n2 1024 --log2n 27 --tamper 128 --n-u 1024 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c5_share.log 2>&1
echo done
