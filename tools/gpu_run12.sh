cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_var22.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1_var -c 1 -o gpurun_out/var_full python bench.py --varlen --mode epoch --n2 1024 --log2n 20 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_ncu_var.log 2>&1
echo done
