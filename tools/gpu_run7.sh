cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for mb in 2 3; do
  POSLO_S1M_MINB=$mb timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_minb$mb.log 2>&1
done
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 26 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_epoch26.log 2>&1
timeout 900 python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_var22.log 2>&1
timeout 900 python bench.py --suite 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_s2.log 2>&1
timeout 1500 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_epoch30.log 2>&1
echo done
