cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for m in 5 6; do
  POSLO_SHA_MODE=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_mode$m.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1 -s 2 -c 1 -o gpurun_out/prof_hash_s1c_m6 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
echo done
