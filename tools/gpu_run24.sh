cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 26 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_epoch26.log 2>&1
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_epoch30.log 2>&1
timeout 900 python bench.py --mode tamper --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_tamper30.log 2>&1
echo done
