# Suite-2 iteration: parity on every suite-2 path, then the suite-2 bench line
# at each CTA size of the persistent kernel, and one ncu capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "suite2 or suite-2 or s2 or 2-" > gpurun_out/s2_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/s2_parity_all.log 2>&1
for t in 512 384 256; do
  POSLO_S2_THREADS=$t timeout 600 python bench.py --suite 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_s2_t$t.json.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_s2 -c 1 -f -o /tmp/k2 python bench.py --suite 2 --log2n 24 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu -i /tmp/k2.ncu-rep --page raw --csv > gpurun_out/ncu_s2p_raw.csv 2>&1
ncu -i /tmp/k2.ncu-rep --page source --csv > gpurun_out/ncu_s2p_source.csv 2>&1
echo done
